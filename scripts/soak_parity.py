"""Soak test: many random mixed gate records (LIN2 with random gate constants
and signs, MUX, majority / XOR3, half adders) on the GPU vs the oracle's or_run_gates,
several levels deep (each level reads the previous level's outputs).
Usage: python scripts/soak_parity.py [records_per_level] [levels]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1806_03461_b200 import tfhe  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
levels = int(sys.argv[2]) if len(sys.argv) > 2 else 3
names = list(tfhe.GATE_LIN)
for unroll in (2, 1):
    p = tfhe.default_params(); p.bk_unroll = unroll
    keys = tfhe.KeySet(seed=2024, params=p)
    op = O.default_params(); op.bk_unroll = unroll
    octx = O.Context(op, O.Keys(op, 2024))
    eng = tfhe.Engine(keys)
    rng = np.random.default_rng(unroll)
    n_in = 256
    total = n_in + levels * 2 * n  # per level: n record outputs + n half-adder XOR outputs
    cts = keys.encrypt(rng.integers(0, 2, n_in).astype(np.uint8), seed=5, stream=9)
    eng.reserve(total)
    eng.upload(0, cts)
    pool = np.zeros((total, op.n + 1), np.uint32)
    pool[:n_in] = cts
    t_gpu = t_cpu = 0.0
    lo = 0
    for lv in range(levels):
        base = n_in + lv * 2 * n
        recs = tfhe.gate_records(n)
        recs["dst"] = base + np.arange(n)
        srcs = rng.integers(lo, base, (n, 3))
        recs["src_a"], recs["src_b"], recs["src_c"] = srcs[:, 0], srcs[:, 1], srcs[:, 2]
        kind = rng.integers(0, 4, n)
        recs["kind"] = kind
        for i in range(n):
            if kind[i] == 0:
                c0, al, be = tfhe.GATE_LIN[names[rng.integers(0, len(names))]]
                recs["c0"][i], recs["alpha"][i], recs["beta"][i] = c0, al, be
            elif kind[i] == 1:
                recs["alpha"][i], recs["beta"][i] = rng.choice((-1, 1)), rng.choice((-1, 1))
            elif kind[i] == 2:
                coef = (-2, -2, -2) if rng.integers(0, 2) else tuple(int(v) for v in rng.choice((-1, 1), 3))
                recs["alpha"][i], recs["beta"][i], recs["gamma"][i] = coef
            else:  # half adder: AND of random literals -> dst, XOR -> base + n + i
                al, be = rng.choice((-1, 1)), rng.choice((-1, 1))
                if recs["src_a"][i] == recs["src_b"][i]:
                    recs["src_b"][i] = lo if recs["src_a"][i] != lo else lo + 1
                recs["c0"][i] = (-(1 << 29)) & 0xFFFFFFFF
                recs["alpha"][i], recs["beta"][i], recs["gamma"][i] = al, be, al * be
                recs["src_c"][i] = base + n + i
        t0 = time.time(); eng.run_gates(recs); eng.sync(); t_gpu += time.time() - t0
        t0 = time.time(); octx.run_gates(recs, pool, threads=os.cpu_count() or 1); t_cpu += time.time() - t0
        lo = base
    got = eng.download(n_in, levels * 2 * n)
    same = np.array_equal(got, pool[n_in:])
    print(f"bk_unroll={unroll}: {levels} levels x {n} records, GPU == oracle word for word: {same} "
          f"(GPU {t_gpu:.2f} s, oracle {t_cpu:.1f} s on {os.cpu_count()} threads)", flush=True)
    eng.close()
