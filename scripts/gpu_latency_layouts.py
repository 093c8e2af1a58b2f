"""Narrow-level latency (one wave of <= #SM bootstraps) for both key layouts
and both narrow-level kernels.  Usage: python scripts/gpu_latency_layouts.py"""
import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CODE = r'''
import sys, json, numpy as np
from paper_1806_03461_b200 import tfhe
unroll = int(sys.argv[1])
p = tfhe.default_params(); p.bk_unroll = unroll
keys = tfhe.KeySet(seed=3, params=p)
eng = tfhe.Engine(keys)
res = {}
for n in (1, 16, 74, 148, 296, 592):
    rng = np.random.default_rng(n)
    a = rng.integers(0, 2, n).astype(np.uint8); b = rng.integers(0, 2, n).astype(np.uint8)
    eng.reserve(3 * n)
    eng.upload(0, np.concatenate([keys.encrypt(a, seed=1, stream=1), keys.encrypt(b, seed=1, stream=2)]))
    recs = tfhe.gate_records(n)
    c0, al, be = tfhe.GATE_LIN["NAND"]
    recs["dst"], recs["src_a"], recs["src_b"] = np.arange(2 * n, 3 * n), np.arange(n), np.arange(n, 2 * n)
    recs["c0"], recs["alpha"], recs["beta"] = c0, al, be
    eng.run_gates(recs); eng.sync()
    ts = []
    for _ in range(5):
        eng.run_gates(recs); ts.append(sum(eng.last_timing()))
    ok = bool(np.array_equal(keys.decrypt(eng.download(2 * n, n)), 1 - (a & b)))
    res[n] = (round(min(ts), 3), ok)
print(json.dumps(res))
'''
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for unroll, lat, clu in ((2, "1", "1"), (2, "1", "0"), (2, "0", "0"), (1, "1", "0"), (1, "0", "0")):
    env = dict(os.environ, HEBNN_B200_LATENCY_MODE=lat, HEBNN_B200_CLUSTER_MODE=clu)
    r = subprocess.run([sys.executable, "-c", CODE, str(unroll)], cwd=root, env=env, capture_output=True, text=True)
    print(f"bk_unroll={unroll} latency_mode={lat} cluster_mode={clu} ms(BR+KS) per level width:",
          r.stdout.strip() or r.stderr[-800:], flush=True)
