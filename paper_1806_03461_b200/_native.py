"""ctypes binding of libhebnn_b200.so (C ABI declared in include/hebnn_b200.h).

The library is built in-tree by ``paper_1806_03461_b200.build`` (nvcc,
sm_100a).  There is no fallback: if the library is missing or a CUDA call
fails the caller gets an exception, never a CPU substitute.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HEBNN_B200_LIB") or os.path.join(_HERE, "_lib", "libhebnn_b200.so")

HB_OK = 0
HB_EINVAL = -1
HB_ECUDA = -2
HB_ENOMEM = -3

GATE_LIN2 = 0
GATE_MUX = 1
GATE_LIN3 = 2
GATE_HA = 3

# Every symbol the header declares (tests check the library exports them all).
EXPORTED = (
    "hb_abi_version", "hb_last_error", "hb_default_params", "hb_params_valid", "hb_lwe_words", "hb_bk_words",
    "hb_ksk_words", "hb_keygen", "hb_encrypt", "hb_phase", "hb_decrypt", "hb_engine_create",
    "hb_engine_destroy", "hb_pool_reserve", "hb_pool_capacity", "hb_pool_stride", "hb_pool_upload",
    "hb_pool_download", "hb_pool_gather", "hb_run_gates", "hb_sync", "hb_last_timing",
    "hb_counters", "hb_debug_blind_rotate", "hb_debug_bootstrap_wo_ks", "hb_debug_keyswitch",
    "hb_debug_fft_margin", "hb_debug_fourier", "hb_flush_l2", "hb_measure_fp64_peak",
    "hb_pool_upload_async", "hb_pool_download_async", "hb_pool_gather_device", "hb_pool_put_device",
)


class NativeLibraryMissing(RuntimeError):
    """libhebnn_b200.so is not built; run paper_1806_03461_b200.build.build()."""


class DeviceError(RuntimeError):
    """A CUDA/driver failure inside the engine (never a user error)."""


class HbParams(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32),
        ("N", ctypes.c_int32),
        ("k", ctypes.c_int32),
        ("bg_bits", ctypes.c_int32),
        ("l", ctypes.c_int32),
        ("ks_base_bits", ctypes.c_int32),
        ("ks_t", ctypes.c_int32),
        ("bk_unroll", ctypes.c_int32),
        ("lwe_stdev", ctypes.c_double),
        ("bk_stdev", ctypes.c_double),
    ]


GATE_DTYPE = np.dtype(
    [("dst", "<u4"), ("src_a", "<u4"), ("src_b", "<u4"), ("src_c", "<u4"), ("c0", "<u4"),
     ("alpha", "i1"), ("beta", "i1"), ("kind", "i1"), ("gamma", "i1")]
)
assert GATE_DTYPE.itemsize == 24


_lib = None


_dag = None


def dag_module():
    """The host gate-DAG extension (csrc/hb_dag.cpp; built by paper_1806_03461_b200.build)."""
    global _dag
    if _dag is None:
        import importlib.util
        import sysconfig

        path = os.path.join(_HERE, "_lib", "hb_dag" + sysconfig.get_config_var("EXT_SUFFIX"))
        if not os.path.exists(path):
            raise NativeLibraryMissing(f"{path} not found: build it with `python -m paper_1806_03461_b200.build`")
        spec = importlib.util.spec_from_file_location("hb_dag", path)
        _dag = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(_dag)
    return _dag


def lib():
    """Load the engine library (raises NativeLibraryMissing if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            f"{LIB_PATH} not found: build it with `python -c 'import paper_1806_03461_b200.build as b; b.build()'`"
        )
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    u32p, vp, sz = P(ctypes.c_uint32), ctypes.c_void_p, ctypes.c_size_t
    sig = {
        "hb_abi_version": ([], ctypes.c_int),
        "hb_last_error": ([], ctypes.c_char_p),
        "hb_default_params": ([P(HbParams)], None),
        "hb_params_valid": ([P(HbParams)], ctypes.c_int),
        "hb_lwe_words": ([P(HbParams)], sz),
        "hb_bk_words": ([P(HbParams)], sz),
        "hb_ksk_words": ([P(HbParams)], sz),
        "hb_keygen": ([P(HbParams), ctypes.c_uint64, u32p, u32p, u32p, u32p, ctypes.c_int], ctypes.c_int),
        "hb_encrypt": ([P(HbParams), u32p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, P(ctypes.c_uint8),
                        sz, u32p, sz],
                       ctypes.c_int),
        "hb_phase": ([P(HbParams), u32p, u32p, sz, sz, P(ctypes.c_int32)], ctypes.c_int),
        "hb_decrypt": ([P(HbParams), u32p, u32p, sz, sz, P(ctypes.c_uint8)], ctypes.c_int),
        "hb_engine_create": ([ctypes.c_int, P(HbParams), u32p, u32p, P(vp)], ctypes.c_int),
        "hb_engine_destroy": ([vp], ctypes.c_int),
        "hb_pool_reserve": ([vp, sz], ctypes.c_int),
        "hb_pool_capacity": ([vp], sz),
        "hb_pool_stride": ([vp], sz),
        "hb_pool_upload": ([vp, sz, sz, u32p, sz], ctypes.c_int),
        "hb_pool_download": ([vp, sz, sz, u32p, sz], ctypes.c_int),
        "hb_pool_gather": ([vp, u32p, sz, u32p, sz], ctypes.c_int),
        "hb_pool_gather_device": ([vp, u32p, sz, vp, sz], ctypes.c_int),
        "hb_pool_put_device": ([vp, sz, sz, vp, sz], ctypes.c_int),
        "hb_pool_upload_async": ([vp, sz, sz, u32p, sz], ctypes.c_int),
        "hb_pool_download_async": ([vp, sz, sz, u32p, sz], ctypes.c_int),
        "hb_run_gates": ([vp, vp, sz, ctypes.c_uint32], ctypes.c_int),
        "hb_sync": ([vp], ctypes.c_int),
        "hb_last_timing": ([vp, P(ctypes.c_float), P(ctypes.c_float)], ctypes.c_int),
        "hb_counters": ([vp, P(ctypes.c_uint64), P(ctypes.c_uint64), P(ctypes.c_uint64)], ctypes.c_int),
        "hb_debug_blind_rotate": ([vp, u32p, ctypes.c_uint32, ctypes.c_int32, u32p], ctypes.c_int),
        "hb_debug_bootstrap_wo_ks": ([vp, u32p, sz, u32p], ctypes.c_int),
        "hb_debug_keyswitch": ([vp, u32p, sz, u32p], ctypes.c_int),
        "hb_debug_fft_margin": ([vp, P(ctypes.c_double)], ctypes.c_int),
        "hb_debug_fourier": ([vp, u32p, sz, P(ctypes.c_double), ctypes.c_int], ctypes.c_int),
        "hb_flush_l2": ([vp, sz], ctypes.c_int),
        "hb_measure_fp64_peak": ([vp, P(ctypes.c_double)], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def check(rc):
    """Map an hb_* status code to an exception."""
    if rc == HB_OK:
        return
    msg = lib().hb_last_error().decode(errors="replace")
    if rc == HB_EINVAL:
        raise ValueError(msg)
    raise DeviceError(f"hebnn_b200 engine error {rc}: {msg}")


def u32p(a):
    assert a.dtype == np.uint32 and a.flags.c_contiguous, (a.dtype, a.flags)
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def default_params():
    p = HbParams()
    lib().hb_default_params(ctypes.byref(p))
    return p
