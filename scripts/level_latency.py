"""Per-level device latency (blind rotation + key switch, ms) by level width
for the default key layout.  Usage: python scripts/level_latency.py
(HEBNN_B200_LIB selects an engine variant)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_03461_b200 import tfhe  # noqa: E402

keys = tfhe.KeySet(seed=3)
eng = tfhe.Engine(keys)
res = {}
for n in (1, 16, 20, 21, 32, 74, 75, 148, 149, 296, 297, 400, 444, 445, 592, 600, 729, 900, 1036, 1184, 4096):
    rng = np.random.default_rng(n)
    a = rng.integers(0, 2, n).astype(np.uint8)
    b = rng.integers(0, 2, n).astype(np.uint8)
    eng.reserve(3 * n)
    eng.upload(0, np.concatenate([keys.encrypt(a, seed=1, stream=1), keys.encrypt(b, seed=1, stream=2)]))
    recs = tfhe.gate_records(n)
    c0, al, be = tfhe.GATE_LIN["NAND"]
    recs["dst"], recs["src_a"], recs["src_b"] = np.arange(2 * n, 3 * n), np.arange(n), np.arange(n, 2 * n)
    recs["c0"], recs["alpha"], recs["beta"] = c0, al, be
    eng.run_gates(recs)
    eng.sync()
    br, ks = [], []
    for _ in range(5):
        eng.run_gates(recs)
        t = eng.last_timing()
        br.append(t[0])
        ks.append(t[1])
    ok = bool(np.array_equal(keys.decrypt(eng.download(2 * n, n)), 1 - (a & b)))
    res[n] = {"br_ms": round(min(br), 3), "ks_ms": round(min(ks), 3), "ok": ok}
print(json.dumps(res))
