"""Narrow-level latency and exactness by kernel: NAND levels of n bootstraps vs the oracle.

    python scripts/narrow_levels.py [n ...]

Prints, per level width, the blind-rotation and key-switch times (CUDA events,
best of 5), plaintext correctness and bit-exactness of three ciphertexts
against the exact-integer oracle (test infrastructure).  Engine switches such as
HEBNN_B200_BINSPLIT select the kernel family.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1806_03461_b200 import tfhe  # noqa: E402
from oracle import oracle as O  # noqa: E402

widths = [int(a) for a in sys.argv[1:]] or [1, 3, 8, 12, 16, 20, 24, 32, 37, 48, 64, 74]
keys = tfhe.KeySet(seed=42)
eng = tfhe.Engine(keys)
p = O.default_params()
octx = O.Context(p, O.Keys(p, 42))
out = {}
for n in widths:
    rng = np.random.default_rng(n)
    a = rng.integers(0, 2, n).astype(np.uint8)
    b = rng.integers(0, 2, n).astype(np.uint8)
    ca, cb = keys.encrypt(a, seed=1, stream=1), keys.encrypt(b, seed=1, stream=2)
    eng.reserve(3 * n)
    eng.upload(0, np.concatenate([ca, cb]))
    recs = tfhe.gate_records(n)
    c0, al, be = tfhe.GATE_LIN["NAND"]
    recs["dst"], recs["src_a"], recs["src_b"] = np.arange(2 * n, 3 * n), np.arange(n), np.arange(n, 2 * n)
    recs["c0"], recs["alpha"], recs["beta"] = c0, al, be
    eng.run_gates(recs)
    eng.sync()
    got = eng.download(2 * n, n)
    ok_bits = bool(np.array_equal(keys.decrypt(got), 1 - (a & b)))
    pick = sorted({0, n // 2, n - 1})
    exact = all(np.array_equal(got[i], octx.gate(c0, al, ca[i], be, cb[i])) for i in pick)
    t = []
    for _ in range(5):
        eng.run_gates(recs)
        t.append(eng.last_timing())
    out[n] = {"bits_ok": ok_bits, "bit_exact_vs_oracle": exact, "br_ms": round(min(x[0] for x in t), 4),
              "ks_ms": round(min(x[1] for x in t), 4)}
    print(n, out[n], flush=True)
print(json.dumps(out))
