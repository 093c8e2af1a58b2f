import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from paper_1806_03461_b200 import tfhe
K = tfhe.KeySet(seed=1); eng = tfhe.Engine(K)
rng = np.random.default_rng(0)
N = 4096
eng.reserve(3 * N)
eng.upload(0, K.encrypt(rng.integers(0, 2, 2 * N).astype(np.uint8), 3, 1))
c0, al, be = tfhe.GATE_LIN["NAND"]
for n in (1, 16, 64, 148, 200, 296, 444, 592, 1184, 2368, 4096):
    recs = tfhe.gate_records(n)
    recs["dst"] = 2 * N + np.arange(n); recs["src_a"] = np.arange(n); recs["src_b"] = N + np.arange(n)
    recs["c0"], recs["alpha"], recs["beta"] = c0, al, be
    eng.run_gates(recs); eng.sync()
    ts = []
    for _ in range(3):
        eng.run_gates(recs); br, ks = eng.last_timing(); ts.append(br + ks)
    t = min(ts)
    print(f"level of {n:5d} gates: {t:7.2f} ms  -> {n / t * 1e3:9.0f} gates/s", flush=True)
