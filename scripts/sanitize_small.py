"""Small engine workload for compute-sanitizer (one tool per gpurun call)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_03461_b200 import tfhe  # noqa: E402

keys = tfhe.KeySet(seed=3)
eng = tfhe.Engine(keys)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rng = np.random.default_rng(0)
a = rng.integers(0, 2, n).astype(np.uint8)
b = rng.integers(0, 2, n).astype(np.uint8)
eng.reserve(4 * n)
eng.upload(0, keys.encrypt(a, seed=1, stream=1))
eng.upload(n, keys.encrypt(b, seed=1, stream=2))
recs = tfhe.gate_records(n)
recs["dst"], recs["src_a"], recs["src_b"] = np.arange(2 * n, 3 * n), np.arange(n), np.arange(n, 2 * n)
recs["src_c"] = np.arange(n)
recs["kind"] = np.arange(n) % 2          # mix LIN2 and MUX records
recs["c0"] = np.where(recs["kind"] == 0, tfhe.GATE_LIN["NAND"][0], 0)
recs["alpha"] = np.where(recs["kind"] == 0, -1, 1)
recs["beta"] = np.where(recs["kind"] == 0, -1, 1)
eng.run_gates(recs)
out = eng.download(2 * n, n)
want = np.where(np.arange(n) % 2 == 0, 1 - (a & b), np.where(a == 1, b, a))  # MUX(a, b, a)
assert np.array_equal(keys.decrypt(out), want), "wrong results"
eng.debug_blind_rotate(keys.encrypt([1], seed=2)[0], iters=5)
eng.debug_keyswitch(np.zeros((3, 1025), np.uint32))
print("sanitize workload ok")
