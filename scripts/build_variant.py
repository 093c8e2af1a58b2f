"""Build an experimental variant of the engine with extra -D flags into
paper_1806_03461_b200/_lib/exp_<name>.so (timing experiments only).
Usage: python scripts/build_variant.py <name> -DFOO=1 [-DBAR=2 ...]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_03461_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(B.HERE, "_lib", f"exp_{name}.so")
cmd = [B.nvcc(), *B.NVCC_FLAGS, *defs, "-o", out, *[os.path.join(B.CSRC, s) for s in B.SOURCES]]
subprocess.run(cmd, check=True)
print(out)
