"""Determinism stress of a blind-rotation variant (engine environment switch).

    python scripts/ws_race.py HEBNN_B200_U2WS [n] [runs]

Runs n mixed gates (default 16,384) `runs` times on the variant and once on the
default kernel, and reports every output ciphertext that differs from the
default kernel's (index, index mod the wave size, differing words).
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_03461_b200 import tfhe  # noqa: E402

var = sys.argv[1] if len(sys.argv) > 1 else "HEBNN_B200_U2WS"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
runs = int(sys.argv[3]) if len(sys.argv) > 3 else 8
params = tfhe.default_params()
params.bk_unroll = int(sys.argv[4]) if len(sys.argv) > 4 else 2
K = tfhe.KeySet(seed=1, params=params)
rng = np.random.default_rng(78)
a = rng.integers(0, 2, n).astype(np.uint8)
b = rng.integers(0, 2, n).astype(np.uint8)
ca, cb = K.encrypt(a, seed=61, stream=1), K.encrypt(b, seed=61, stream=2)
recs = tfhe.gate_records(n)
kinds = list(tfhe.GATE_LIN)
pick = rng.integers(0, len(kinds), n)
for k, name in enumerate(kinds):
    c0, al, be = tfhe.GATE_LIN[name]
    sel = pick == k
    recs["c0"][sel], recs["alpha"][sel], recs["beta"][sel] = c0, al, be
recs["dst"], recs["src_a"], recs["src_b"] = 2 * n + np.arange(n), np.arange(n), n + np.arange(n)


def run(v, count):
    os.environ[var] = v
    eng = tfhe.Engine(K)
    eng.reserve(3 * n)
    eng.upload(0, ca)
    eng.upload(n, cb)
    outs = []
    for _ in range(count):
        eng.run_gates(recs)
        outs.append(eng.download(2 * n, n))
    eng.close()
    return outs


ref = run("0", 1)[0]
bad_total = 0
for i, out in enumerate(run("1", runs)):
    diff = np.nonzero((out != ref).any(axis=1))[0]
    bad_total += diff.size
    words = [int((out[d] != ref[d]).sum()) for d in diff[:8]]
    print(f"run {i}: {diff.size} ciphertexts differ; first {diff[:8].tolist()} (mod 592: {(diff[:8] % 592).tolist()}, "
          f"words differing {words})", flush=True)
print("total differing:", bad_total)
