import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from paper_1806_03461_b200 import tfhe
K = tfhe.KeySet(seed=1)
eng = tfhe.Engine(K)
n = 4096
rng = np.random.default_rng(0)
a = rng.integers(0,2,n).astype(np.uint8); b = rng.integers(0,2,n).astype(np.uint8)
eng.reserve(3*n)
eng.upload(0, K.encrypt(a, 3, 1)); eng.upload(n, K.encrypt(b, 3, 2))
recs = tfhe.gate_records(n)
c0, al, be = tfhe.GATE_LIN["NAND"]
recs["dst"] = np.arange(2*n, 3*n); recs["src_a"] = np.arange(n); recs["src_b"] = np.arange(n, 2*n)
recs["c0"] = c0; recs["alpha"] = al; recs["beta"] = be
for it in range(4):
    t = time.time(); eng.run_gates(recs); eng.sync(); dt = time.time() - t
    br, ks = eng.last_timing()
    print(f"iter {it}: wall {dt*1e3:.1f} ms  br {br:.1f} ms ks {ks:.1f} ms  -> {n/dt:.0f} gates/s (br-only {n/br*1e3:.0f}/s)", flush=True)
out = eng.download(2*n, n)
print("nand correct:", np.array_equal(K.decrypt(out), 1 - (a & b)))
