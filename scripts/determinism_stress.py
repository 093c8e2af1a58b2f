"""Run the same batch of bootstraps repeatedly and check the outputs are
identical every time (a race in a kernel would show up as a difference) and
the FFT rounding margin stays small.  Usage: python scripts/determinism_stress.py [reps] [count]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1806_03461_b200 import tfhe  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
count = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
for unroll in (1, 2):
    p = tfhe.default_params(); p.bk_unroll = unroll
    keys = tfhe.KeySet(seed=77, params=p)
    eng = tfhe.Engine(keys)
    rng = np.random.default_rng(unroll)
    lin = keys.encrypt(rng.integers(0, 2, count).astype(np.uint8), seed=9, stream=0)
    lin[count // 2:] = rng.integers(0, 2 ** 32, (count - count // 2, lin.shape[1]), dtype=np.uint64).astype(np.uint32)
    ref = eng.debug_bootstrap_wo_ks(lin)
    margins, bad = [eng.debug_fft_margin()], 0
    for r in range(reps):
        out = eng.debug_bootstrap_wo_ks(lin)
        margins.append(eng.debug_fft_margin())
        if not np.array_equal(out, ref):
            rows = np.flatnonzero((out != ref).any(axis=1))
            bad += 1
            print(f"  bk_unroll={unroll} rep {r}: {rows.size} bootstraps differ, e.g. {rows[:5].tolist()}", flush=True)
    print(f"bk_unroll={unroll}: {reps + 1} runs x {count} bootstraps, runs differing from the first: {bad}; "
          f"margin max {max(margins):.4f} min {min(margins):.4f}", flush=True)
    eng.close()

# production kernels (run_gates, wide levels): identical outputs over many repetitions
reps2 = int(os.environ.get("HB_STRESS_REPS", "300"))
for unroll in (2, 1):
    p = tfhe.default_params(); p.bk_unroll = unroll
    keys = tfhe.KeySet(seed=78, params=p)
    eng = tfhe.Engine(keys)
    n = 4096
    rng = np.random.default_rng(10 + unroll)
    eng.reserve(3 * n)
    eng.upload(0, keys.encrypt(rng.integers(0, 2, 2 * n).astype(np.uint8), seed=3, stream=1))
    recs = tfhe.gate_records(n)
    recs["dst"], recs["src_a"], recs["src_b"] = np.arange(2 * n, 3 * n), np.arange(n), np.arange(n, 2 * n)
    c0, al, be = tfhe.GATE_LIN["NAND"]
    recs["c0"], recs["alpha"], recs["beta"] = c0, al, be
    eng.run_gates(recs)
    ref = eng.download(2 * n, n)
    bad = 0
    for r in range(reps2):
        eng.run_gates(recs)
        if r % 50 == 49 or r == reps2 - 1:
            out = eng.download(2 * n, n)
            if not np.array_equal(out, ref):
                bad += 1
                print(f"  bk_unroll={unroll}: outputs differ after rep {r}", flush=True)
    print(f"bk_unroll={unroll}: {reps2} levels of {n} NANDs, checkpoints differing: {bad}", flush=True)
    eng.close()
