"""Largest FFT rounding error |x - round(x)| over many bootstraps (exactness
needs < 0.5), for both key layouts.  Usage: python scripts/fft_margin.py [count]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1806_03461_b200 import tfhe  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
for unroll in (2, 1):
    p = tfhe.default_params(); p.bk_unroll = unroll
    keys = tfhe.KeySet(seed=77, params=p)
    eng = tfhe.Engine(keys)
    rng = np.random.default_rng(unroll)
    worst = 0.0
    for rep in range(4):
        # random linear combinations: fresh encryptions and uniformly random LWE samples
        lin = keys.encrypt(rng.integers(0, 2, count).astype(np.uint8), seed=9, stream=rep)
        lin[count // 2:] = rng.integers(0, 2 ** 32, (count - count // 2, lin.shape[1]), dtype=np.uint64).astype(np.uint32)
        eng.debug_bootstrap_wo_ks(lin)
        worst = max(worst, eng.debug_fft_margin())
    print(f"bk_unroll={unroll}: max |x - round(x)| over {4 * count} bootstraps "
          f"({4 * count * (315 if unroll == 2 else 630)} external products) = {worst:.4f}", flush=True)
    eng.close()
