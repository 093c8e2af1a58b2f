"""GPU parity: every stage of the CUDA gate bootstrap against the exact CPU
oracle on the same seeded keys and inputs (bit-exact ciphertexts)."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_1806_03461_b200 import tfhe

pytestmark = pytest.mark.gpu

P = O.default_params()


@pytest.fixture(params=["pairs", "cggi"])
def kit(request):
    """(engine, keys, oracle context) of one bootstrapping-key layout:
    key pairs (bk_unroll 2, default) or CGGI (bk_unroll 1)."""
    sfx = "" if request.param == "pairs" else "1"
    return tuple(request.getfixturevalue(name + sfx) for name in ("engine", "keys", "octx"))


def _lin(keys, seed, count):
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2, count).astype(np.uint8)
    return keys.encrypt(bits, seed=seed, stream=1)


@pytest.mark.parametrize("iters", [1, 2, 7, 10])
def test_blind_rotate_prefix_bit_exact(kit, iters):
    engine, keys, octx = kit
    lwe = _lin(keys, 11, 1)[0]
    got = engine.debug_blind_rotate(lwe, iters=iters)
    want = octx.blind_rotate(lwe, iters=iters)
    assert np.array_equal(got, want)


def test_bootstrap_wo_ks_bit_exact(kit):
    engine, keys, octx = kit
    lin = _lin(keys, 12, 6)
    got = engine.debug_bootstrap_wo_ks(lin)
    margin = engine.debug_fft_margin()
    for i in range(lin.shape[0]):
        assert np.array_equal(got[i], octx.bootstrap_wo_ks(lin[i]))
    assert margin < 0.25, margin


def test_keyswitch_bit_exact(kit):
    engine, keys, octx = kit
    rng = np.random.default_rng(13)
    big = rng.integers(0, 2**32, (40, P.N + 1), dtype=np.uint64).astype(np.uint32)
    got = engine.debug_keyswitch(big)
    for i in range(big.shape[0]):
        assert np.array_equal(got[i], octx.keyswitch(big[i]))


@pytest.mark.parametrize("name", list(tfhe.GATE_LIN))
def test_gate_truth_table_and_bit_exact(kit, name):
    engine, keys, octx = kit
    c0, al, be = tfhe.GATE_LIN[name]
    a_bits = np.array([0, 0, 1, 1], np.uint8)
    b_bits = np.array([0, 1, 0, 1], np.uint8)
    ca = keys.encrypt(a_bits, seed=21, stream=1)
    cb = keys.encrypt(b_bits, seed=21, stream=2)
    engine.reserve(12)
    engine.upload(0, ca)
    engine.upload(4, cb)
    recs = tfhe.gate_records(4)
    for i in range(4):
        recs[i] = (8 + i, i, 4 + i, 0, c0, al, be, 0, 0)
    engine.run_gates(recs)
    out = engine.download(8, 4)
    fn = {"AND": np.bitwise_and, "OR": np.bitwise_or, "XOR": np.bitwise_xor}
    plain = {
        "AND": a_bits & b_bits, "OR": a_bits | b_bits, "XOR": a_bits ^ b_bits,
        "XNOR": 1 - (a_bits ^ b_bits), "NAND": 1 - (a_bits & b_bits), "NOR": 1 - (a_bits | b_bits),
    }[name]
    assert np.array_equal(keys.decrypt(out), plain)
    for i in range(4):
        assert np.array_equal(out[i], octx.gate(c0, al, ca[i], be, cb[i]))


def test_mux_bit_exact(kit):
    engine, keys, octx = kit
    s = np.array([0, 0, 0, 0, 1, 1, 1, 1], np.uint8)
    a = np.array([0, 0, 1, 1, 0, 0, 1, 1], np.uint8)
    b = np.array([0, 1, 0, 1, 0, 1, 0, 1], np.uint8)
    cs, ca, cb = (keys.encrypt(v, seed=31, stream=k) for k, v in enumerate((s, a, b)))
    engine.reserve(32)
    engine.upload(0, cs)
    engine.upload(8, ca)
    engine.upload(16, cb)
    recs = tfhe.gate_records(8)
    for i in range(8):
        recs[i] = (24 + i, i, 8 + i, 16 + i, 0, 1, 1, 1, 0)
    engine.run_gates(recs)
    out = engine.download(24, 8)
    assert np.array_equal(keys.decrypt(out), np.where(s == 1, a, b))
    for i in (0, 5):
        assert np.array_equal(out[i], octx.mux(cs[i], ca[i], cb[i]))


@pytest.mark.parametrize("name", ["MAJ", "XOR3", "MAJ_NEG"])
def test_three_input_gates_truth_table_and_bit_exact(kit, name):
    """hb_gate LIN3: majority (a full adder's carry) and 3-input XOR (its sum)
    in one bootstrap each, bit-exact vs the oracle's or_gate3."""
    engine, keys, octx = kit
    bits = np.array([[(i >> k) & 1 for k in range(3)] for i in range(8)], np.uint8).T  # [3][8]
    cts = [keys.encrypt(bits[k], seed=41, stream=k) for k in range(3)]
    engine.reserve(32)
    for k in range(3):
        engine.upload(8 * k, cts[k])
    coef = {"MAJ": (1, 1, 1), "XOR3": (-2, -2, -2), "MAJ_NEG": (1, -1, 1)}[name]
    recs = tfhe.gate_records(8)
    for i in range(8):
        recs[i] = (24 + i, i, 8 + i, 16 + i, 0, coef[0], coef[1], 2, coef[2])
    engine.run_gates(recs)
    out = engine.download(24, 8)
    a, b, c = bits.astype(int)
    want = {"MAJ": (a + b + c) >= 2, "XOR3": (a ^ b ^ c) == 1, "MAJ_NEG": (a + (1 - b) + c) >= 2}[name]
    assert np.array_equal(keys.decrypt(out), want.astype(np.uint8))
    for i in (0, 3, 5, 7):
        assert np.array_equal(out[i], octx.gate3(0, coef[0], cts[0][i], coef[1], cts[1][i], coef[2], cts[2][i]))


def test_gpu_matches_committed_golden_vectors(kit):
    """The sm_100a engine reproduces tests/golden/tfhe_golden_seed42.npz (CGGI)
    and tfhe_golden_pairs_seed42.npz (key pairs) — oracle-generated: keys from
    seed 42, encryptions, gates, MUX, stages."""
    import os

    engine, keys, _ = kit
    pairs = keys.params.bk_unroll == 2
    name = "tfhe_golden_pairs_seed42.npz" if pairs else "tfhe_golden_seed42.npz"
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", name))
    assert np.array_equal(keys.lwe_key, g["lwe_key"])
    assert int(g["bk_sum"]) == int(keys.bk.astype(np.uint64).sum())
    inputs = g["inputs"]
    assert np.array_equal(keys.encrypt(g["input_bits"], seed=42, stream=77), inputs)
    assert np.array_equal(engine.debug_blind_rotate(inputs[0], iters=4 if pairs else 3), g["acc_prefix3"])
    assert np.array_equal(engine.debug_bootstrap_wo_ks(inputs[2:3])[0], g["bootstrap_wo_ks"])
    assert np.array_equal(engine.debug_keyswitch(g["ks_in"][None, :])[0], g["ks_out"])
    engine.reserve(16)
    engine.upload(0, inputs)
    recs = tfhe.gate_records(len(tfhe.GATE_LIN) + 2)
    names = list(tfhe.GATE_LIN)
    for i, name in enumerate(names):
        c0, al, be = tfhe.GATE_LIN[name]
        recs[i] = (8 + i, 0, 1, 0, c0, al, be, 0, 0)
    recs[len(names)] = (8 + len(names), 1, 0, 4, 0, 1, 1, 1, 0)        # mux(in1, in0, in4)
    recs[len(names) + 1] = (9 + len(names), 0, 2, 1, 0, 1, 1, 1, 0)    # mux(in0, in2, in1)
    engine.run_gates(recs)
    out = engine.download(8, len(names) + 2)
    for i, name in enumerate(names):
        assert np.array_equal(out[i], g[f"gate_{name}"]), name
    assert np.array_equal(out[len(names)], g["mux_010"])
    assert np.array_equal(out[len(names) + 1], g["mux_110"])


def test_wide_level_split_into_chunks_is_identical(keys):
    """hb_run_gates splits levels wider than the work limit into several
    launches; the result must not depend on the split."""
    import os
    import subprocess
    import sys

    code = r'''
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_1806_03461_b200 import tfhe
keys = tfhe.KeySet(seed=42)
eng = tfhe.Engine(keys)
n = 300
rng = np.random.default_rng(4)
eng.reserve(3 * n)
eng.upload(0, keys.encrypt(rng.integers(0, 2, 2 * n).astype(np.uint8), seed=6, stream=1))
recs = tfhe.gate_records(n)
recs["dst"], recs["src_a"], recs["src_b"] = np.arange(2 * n, 3 * n), np.arange(n), np.arange(n, 2 * n)
recs["kind"] = np.where(np.arange(n) % 3 == 0, 1, 0)
recs["src_c"] = (np.arange(n) + 7) % n
recs["c0"], recs["alpha"], recs["beta"] = tfhe.GATE_LIN["XOR"][0], 2, 2
recs["alpha"][recs["kind"] == 1] = 1
recs["beta"][recs["kind"] == 1] = 1
recs["c0"][recs["kind"] == 1] = 0
eng.run_gates(recs)
np.save(sys.argv[1], eng.download(2 * n, n))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for mw in ("0", "64"):
        path = f"/tmp/hb_chunk_{mw}.npy"
        env = dict(os.environ)
        if mw != "0":
            env["HEBNN_B200_MAX_WORK"] = mw
        subprocess.run([sys.executable, "-c", code, path], check=True, cwd=root, env=env)
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("n", [1, 5, 12, 20, 30, 100, 200, 400, 700])
def test_narrow_level_kernels_agree(n):
    """Narrow key-pair levels run, by width, on the 8-CTA bin-split kernel, the
    6-CTA row-split cluster kernel, the 4-CTA bin-split kernel, the 2-CTA
    cluster kernel, the latency kernel or 1-3 bootstraps per CTA; switching
    the narrower kernels off moves a level to the next one.  Every choice must
    give the same ciphertexts (both key layouts), and the default equals the
    oracle's.  400 runs on 3-bootstrap CTAs, 700 as one full wave of
    4-bootstrap CTAs plus a 3-bootstrap remainder launch (split waves) or two
    4-bootstrap waves."""
    import os
    import subprocess
    import sys

    code = r'''
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_1806_03461_b200 import tfhe
n, unroll = int(sys.argv[2]), int(sys.argv[3])
p = tfhe.default_params(); p.bk_unroll = unroll
keys = tfhe.KeySet(seed=42, params=p)
eng = tfhe.Engine(keys)
rng = np.random.default_rng(n)
eng.reserve(4 * n)
eng.upload(0, keys.encrypt(rng.integers(0, 2, 3 * n).astype(np.uint8), seed=6, stream=1))
recs = tfhe.gate_records(n)
recs["dst"], recs["src_a"], recs["src_b"], recs["src_c"] = np.arange(3 * n, 4 * n), np.arange(n), np.arange(n, 2 * n), np.arange(2 * n, 3 * n)
recs["kind"] = np.where(np.arange(n) % 2 == 0, 2, 0)   # MAJ and XOR
recs["alpha"], recs["beta"], recs["gamma"] = 1, 1, 1
recs["c0"] = np.where(recs["kind"] == 2, 0, tfhe.GATE_LIN["XOR"][0])
recs["alpha"][recs["kind"] == 0] = 2
recs["beta"][recs["kind"] == 0] = 2
recs["gamma"][recs["kind"] == 0] = 0
eng.run_gates(recs)
np.save(sys.argv[1], eng.download(3 * n, n))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for unroll in (2, 1):
        outs = []
        # the cluster / bin-split / split-wave switches only select key-pair kernels: the CGGI
        # layout has the latency kernel on or off
        combos = ((("1", "1", "1", "1", "1"), ("1", "1", "0", "1", "1"), ("1", "1", "0", "0", "0"),
                   ("1", "0", "0", "0", "0"), ("0", "0", "0", "0", "0")) if unroll == 2
                  else (("1", "1", "1", "1", "1"), ("0", "0", "0", "0", "0")))
        for lat, clu, bs, c6, sw in combos:
            path = f"/tmp/hb_narrow_{n}_{unroll}_{lat}{clu}{bs}{c6}{sw}.npy"
            env = dict(os.environ, HEBNN_B200_LATENCY_MODE=lat, HEBNN_B200_CLUSTER_MODE=clu, HEBNN_B200_BINSPLIT=bs,
                       HEBNN_B200_CLU6=c6, HEBNN_B200_SPLIT_WAVES=sw)
            subprocess.run([sys.executable, "-c", code, path, str(n), str(unroll)], check=True, cwd=root, env=env)
            outs.append(np.load(path))
        for k in range(1, len(outs)):
            assert np.array_equal(outs[0], outs[k]), (unroll, k)
        # the default path against the exact oracle on two records (a MAJ and an XOR)
        p = tfhe.default_params()
        p.bk_unroll = unroll
        keys = tfhe.KeySet(seed=42, params=p)
        cts = keys.encrypt(np.random.default_rng(n).integers(0, 2, 3 * n).astype(np.uint8), seed=6, stream=1)
        po = O.default_params()
        po.bk_unroll = unroll
        octx = O.Context(po, O.Keys(po, 42))
        for i in range(min(n, 2)):
            if i % 2 == 0:
                want = octx.gate3(0, 1, cts[i], 1, cts[n + i], 1, cts[2 * n + i])
            else:
                want = octx.gate(tfhe.GATE_LIN["XOR"][0], 2, cts[i], 2, cts[n + i])
            assert np.array_equal(outs[0][i], want), (unroll, i)


def test_random_mixed_level_bit_exact_vs_oracle(kit):
    """512 random records of every kind (LIN2 gates with random signs, MUX,
    3-input majority / XOR3 with random signs) in one level: the GPU pool
    equals the oracle's or_run_gates pool word for word."""
    engine, keys, octx = kit
    rng = np.random.default_rng(99)
    n_in, n = 96, 512
    bits = rng.integers(0, 2, n_in).astype(np.uint8)
    cts = keys.encrypt(bits, seed=77, stream=5)
    recs = tfhe.gate_records(n)
    recs["dst"] = n_in + np.arange(n)
    srcs = rng.integers(0, n_in, (n, 3))
    recs["src_a"], recs["src_b"], recs["src_c"] = srcs[:, 0], srcs[:, 1], srcs[:, 2]
    kind = rng.integers(0, 3, n)
    recs["kind"] = kind
    names = list(tfhe.GATE_LIN)
    for i in range(n):
        if kind[i] == 0:
            c0, al, be = tfhe.GATE_LIN[names[rng.integers(0, len(names))]]
            recs["c0"][i], recs["alpha"][i], recs["beta"][i], recs["gamma"][i] = c0, al, be, 0
        elif kind[i] == 1:
            recs["c0"][i], recs["alpha"][i], recs["beta"][i], recs["gamma"][i] = 0, rng.choice((-1, 1)), rng.choice((-1, 1)), 0
        else:
            sg = rng.choice((-1, 1), 3)
            coef = (-2, -2, -2) if rng.integers(0, 2) else tuple(int(v) for v in sg)
            recs["c0"][i], recs["alpha"][i], recs["beta"][i], recs["gamma"][i] = 0, coef[0], coef[1], coef[2]
    engine.reserve(n_in + n)
    engine.upload(0, cts)
    engine.run_gates(recs)
    got = engine.download(n_in, n)
    pool = np.zeros((n_in + n, P.n + 1), np.uint32)
    pool[:n_in] = cts
    import os

    octx.run_gates(recs, pool, threads=os.cpu_count() or 1)
    assert np.array_equal(got, pool[n_in:])
