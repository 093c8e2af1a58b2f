"""One level of n NAND bootstraps (for ncu captures of the narrow-level kernels).
Usage: python scripts/narrow_level.py n [repeats]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_03461_b200 import tfhe  # noqa: E402

n = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
keys = tfhe.KeySet(seed=3)
eng = tfhe.Engine(keys)
rng = np.random.default_rng(n)
a, b = rng.integers(0, 2, n).astype(np.uint8), rng.integers(0, 2, n).astype(np.uint8)
eng.reserve(3 * n)
eng.upload(0, np.concatenate([keys.encrypt(a, seed=1, stream=1), keys.encrypt(b, seed=1, stream=2)]))
recs = tfhe.gate_records(n)
c0, al, be = tfhe.GATE_LIN["NAND"]
recs["dst"], recs["src_a"], recs["src_b"] = np.arange(2 * n, 3 * n), np.arange(n), np.arange(n, 2 * n)
recs["c0"], recs["alpha"], recs["beta"] = c0, al, be
for _ in range(reps):
    eng.run_gates(recs)
eng.sync()
print(n, "ok", bool(np.array_equal(keys.decrypt(eng.download(2 * n, n)), 1 - (a & b))), eng.last_timing())
