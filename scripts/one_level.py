"""One level of n NAND gates (default key layout), 3 launches; for ncu.
Usage: python scripts/one_level.py [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1806_03461_b200 import tfhe

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
keys = tfhe.KeySet(seed=3)
eng = tfhe.Engine(keys)
rng = np.random.default_rng(n)
a = rng.integers(0, 2, n).astype(np.uint8); b = rng.integers(0, 2, n).astype(np.uint8)
eng.reserve(3 * n)
eng.upload(0, np.concatenate([keys.encrypt(a, seed=1, stream=1), keys.encrypt(b, seed=1, stream=2)]))
recs = tfhe.gate_records(n)
c0, al, be = tfhe.GATE_LIN["NAND"]
recs["dst"], recs["src_a"], recs["src_b"] = np.arange(2 * n, 3 * n), np.arange(n), np.arange(n, 2 * n)
recs["c0"], recs["alpha"], recs["beta"] = c0, al, be
for _ in range(3):
    eng.run_gates(recs)
eng.sync()
print("ok", bool(np.array_equal(keys.decrypt(eng.download(2 * n, n)), 1 - (a & b))), eng.last_timing())
