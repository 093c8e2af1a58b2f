"""Find the bootstrap with the largest FFT rounding error (CGGI key) and compare
its output with the exact oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1806_03461_b200 import tfhe  # noqa: E402

unroll = int(sys.argv[1]) if len(sys.argv) > 1 else 1
p = tfhe.default_params(); p.bk_unroll = unroll
keys = tfhe.KeySet(seed=77, params=p)
op = O.default_params(); op.bk_unroll = unroll
octx = O.Context(op, O.Keys(op, 77))
eng = tfhe.Engine(keys)
rng = np.random.default_rng(unroll)
count = 4096
found = []
for rep in range(4):
    lin = keys.encrypt(rng.integers(0, 2, count).astype(np.uint8), seed=9, stream=rep)
    lin[count // 2:] = rng.integers(0, 2 ** 32, (count - count // 2, lin.shape[1]), dtype=np.uint64).astype(np.uint32)
    eng.debug_bootstrap_wo_ks(lin)
    if eng.debug_fft_margin() < 0.2:
        continue
    # bisect by batches of 64
    cand = np.arange(count)
    while cand.size > 1:
        half = cand[: cand.size // 2]
        eng.debug_bootstrap_wo_ks(lin[half])
        cand = half if eng.debug_fft_margin() >= 0.2 else cand[cand.size // 2:]
    i = int(cand[0])
    eng.debug_bootstrap_wo_ks(lin[i:i + 1])
    m = eng.debug_fft_margin()
    got = eng.debug_bootstrap_wo_ks(lin[i:i + 1])[0]
    want = octx.bootstrap_wo_ks(lin[i])
    diff = np.flatnonzero(got != want)
    print(f"rep {rep}: bootstrap {i} margin {m:.4f}; differs from the oracle in {diff.size} coefficients "
          f"{diff[:8].tolist()} (random LWE: {i >= count // 2})", flush=True)
    found.append(i)
print("done", found)
