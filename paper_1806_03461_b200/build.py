"""In-tree build of libhebnn_b200.so (nvcc, sm_100a only).

    python -m paper_1806_03461_b200.build

The shared library lands in paper_1806_03461_b200/_lib/ so it travels with the
repository snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib", "libhebnn_b200.so")
SOURCES = ("hb_host.cpp", "hb_engine.cu")
HEADERS = ("hb_internal.h", "hb_dev_fft.cuh", "hb_br_cggi.cuh", "hb_br_u2.cuh", "hb_br_clu6.cuh", "hb_br_binsplit.cuh", "hb_ks.cuh")

NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
    "-shared",
]


def nvcc():
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found")
    return path


def _stale():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "hebnn_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def dag_out():
    import sysconfig

    return os.path.join(HERE, "_lib", "hb_dag" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_dag(force=False):
    """The host gate-DAG extension (CPython + numpy C API, g++): csrc/hb_dag.cpp -> _lib/hb_dag*.so."""
    import sysconfig

    import numpy

    out, src = dag_out(), os.path.join(CSRC, "hb_dag.cpp")
    if not force and os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(src),
                                                                          os.path.getmtime(__file__)):
        return out
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cxx = shutil.which("g++") or "g++"
    cmd = [cxx, "-O2", "-std=c++17", "-shared", "-fPIC", "-fvisibility=hidden",
           "-I", numpy.get_include(), "-I", sysconfig.get_paths()["include"], src, "-o", out + ".tmp"]
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


def build(force=False, verbose=False):
    build_dag(force)
    if not force and not _stale():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    tmp = OUT + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, "-o", tmp, *[os.path.join(CSRC, s) for s in SOURCES]]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
