"""Key-pair bootstrapping key (bk_unroll 2) on the GPU vs the oracle, and
throughput of both key layouts.  Usage: python scripts/gpu_u2_check.py"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_1806_03461_b200 import tfhe

for unroll in (2, 1):
    p = tfhe.default_params(); p.bk_unroll = unroll
    keys = tfhe.KeySet(seed=7, params=p)
    op = O.default_params(); op.bk_unroll = unroll
    ok_ = O.Keys(op, 7)
    same_keys = np.array_equal(keys.bk.reshape(-1), ok_.bk.reshape(-1)) and np.array_equal(keys.ksk.reshape(-1), ok_.ksk.reshape(-1))
    octx = O.Context(op, ok_)
    eng = tfhe.Engine(keys)
    rng = np.random.default_rng(1)
    lwe = O.encrypt(op, ok_, np.array([1], np.uint8), 7, 3)[0]
    res = {}
    for iters in (2, 4, 10, -1):
        g = eng.debug_blind_rotate(lwe, iters=iters)
        o = octx.blind_rotate(lwe, iters=iters)
        res[iters] = bool(np.array_equal(np.asarray(g).reshape(-1), np.asarray(o).reshape(-1)))
    lin = O.encrypt(op, ok_, rng.integers(0, 2, 64).astype(np.uint8), 7, 4)
    gb = eng.debug_bootstrap_wo_ks(lin)
    margin = eng.debug_fft_margin()
    ob = np.array([octx.bootstrap_wo_ks(lin[i]) for i in range(8)])
    bs_ok = bool(np.array_equal(np.asarray(gb)[:8], ob))
    # throughput: 4096 NANDs
    n = 4096
    a = rng.integers(0, 2, n).astype(np.uint8); b = rng.integers(0, 2, n).astype(np.uint8)
    cts = np.concatenate([keys.encrypt(a, seed=1, stream=1), keys.encrypt(b, seed=1, stream=2)])
    eng.reserve(3 * n); eng.upload(0, cts)
    recs = tfhe.gate_records(n)
    c0, al, be = tfhe.GATE_LIN["NAND"]
    recs["dst"], recs["src_a"], recs["src_b"] = np.arange(2 * n, 3 * n), np.arange(n), np.arange(n, 2 * n)
    recs["c0"], recs["alpha"], recs["beta"] = c0, al, be
    eng.run_gates(recs); eng.sync()
    ts = []
    for _ in range(5):
        eng.run_gates(recs); ts.append(eng.last_timing())
    out = eng.download(2 * n, n)
    correct = bool(np.array_equal(keys.decrypt(out), 1 - (a & b)))
    # oracle parity of a few full gates
    sub = np.arange(0, n, 512)
    og = np.array([octx.gate(c0, al, cts[i], be, cts[n + i]) for i in sub])
    gate_ok = bool(np.array_equal(out[sub], og))
    ph = keys.phase(out).astype(np.int64)
    err = np.abs(ph - np.where(1 - (a & b), 1 << 29, -(1 << 29)))
    br = min(t[0] for t in ts); ks = min(t[1] for t in ts)
    print(f"unroll={unroll} keys_match_oracle={same_keys} blind_rotate_parity={res} bootstrap_parity={bs_ok} "
          f"gate_parity={gate_ok} fft_margin={margin:.4f} correct={correct} "
          f"noise_rms=2^{np.log2(np.sqrt((err.astype(float)**2).mean())/2**32):.2f} max=2^{np.log2(err.max()/2**32):.2f} "
          f"BR {br:.2f} ms KS {ks:.2f} ms -> {n / (br + ks) * 1e3:.0f} gates/s", flush=True)
    eng.close()
