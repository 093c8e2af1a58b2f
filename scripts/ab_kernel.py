"""A/B of wide-level blind-rotation variants selected by engine environment switches.

    python scripts/ab_kernel.py HEBNN_B200_U2WS [n_gates] [bk_unroll]

Runs the same level of n NAND gates (default 4,096) with the switch 0 and 1 on
fresh engines of one key set, reports the blind-rotation / key-switch times
(CUDA events on the engine stream, median of 7) and checks that both variants
produce identical ciphertexts and the right plaintexts.
"""

import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_03461_b200 import tfhe  # noqa: E402

var = sys.argv[1] if len(sys.argv) > 1 else "HEBNN_B200_U2WS"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
unroll = int(sys.argv[3]) if len(sys.argv) > 3 else 2
params = tfhe.default_params()
params.bk_unroll = unroll
K = tfhe.KeySet(seed=1, params=params)
rng = np.random.default_rng(0)
a = rng.integers(0, 2, n).astype(np.uint8)
b = rng.integers(0, 2, n).astype(np.uint8)
ca, cb = K.encrypt(a, 3, 1), K.encrypt(b, 3, 2)
recs = tfhe.gate_records(n)
c0, al, be = tfhe.GATE_LIN["NAND"]
recs["dst"] = np.arange(2 * n, 3 * n)
recs["src_a"] = np.arange(n)
recs["src_b"] = np.arange(n, 2 * n)
recs["c0"], recs["alpha"], recs["beta"] = c0, al, be
outs = {}
for v in ("0", "1"):
    os.environ[var] = v
    eng = tfhe.Engine(K)
    eng.reserve(3 * n)
    eng.upload(0, ca)
    eng.upload(n, cb)
    eng.run_gates(recs)
    eng.sync()
    brs, kss = [], []
    for _ in range(7):
        eng.run_gates(recs)
        eng.sync()
        br, ks = eng.last_timing()
        brs.append(br)
        kss.append(ks)
    out = eng.download(2 * n, n)
    outs[v] = out
    ok = np.array_equal(K.decrypt(out), 1 - (a & b))
    br, ks = statistics.median(brs), statistics.median(kss)
    print(f"{var}={v}: blind rotation {br:.3f} ms  key switch {ks:.3f} ms  -> {n / (br + ks) * 1e3:.0f} gates/s  "
          f"plaintexts ok: {ok}", flush=True)
    eng.close()
print("identical ciphertexts:", np.array_equal(outs["0"], outs["1"]))
if os.environ.get("AB_OUT"):  # cross-library comparisons (HEBNN_B200_LIB variants)
    np.save(os.environ["AB_OUT"], outs["1"])
