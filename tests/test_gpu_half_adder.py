"""GPU parity of the half-adder record (hb_gate kind HA: one blind rotation,
two extractions, two key switches) against the exact CPU oracle
(oracle/tfhe_oracle.c or_half_adder), on every blind-rotation kernel path and
both key layouts, plus its phase noise against the budget."""

import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1806_03461_b200 import tfhe
from paper_1806_03461_b200._native import GATE_HA

pytestmark = pytest.mark.gpu

P = O.default_params()
EIGHTH = 1 << 29


def _ha_records(rng, n, n_in, base):
    """n HA records on random input pairs with random literal signs; outputs
    AND -> base + i, XOR -> base + n + i."""
    recs = tfhe.gate_records(n)
    src = np.stack([rng.choice(n_in, 2, replace=False) for _ in range(n)])
    recs["src_a"], recs["src_b"] = src[:, 0], src[:, 1]
    recs["alpha"] = rng.choice((-1, 1), n)
    recs["beta"] = rng.choice((-1, 1), n)
    recs["gamma"] = recs["alpha"] * recs["beta"]
    recs["c0"] = (-EIGHTH) & 0xFFFFFFFF
    recs["kind"] = GATE_HA
    recs["dst"] = base + np.arange(n)
    recs["src_c"] = base + n + np.arange(n)
    return recs


@pytest.fixture(params=["pairs", "cggi"])
def kit(request):
    sfx = "" if request.param == "pairs" else "1"
    return tuple(request.getfixturevalue(name + sfx) for name in ("engine", "keys", "octx"))


@pytest.mark.parametrize("n", [1, 40, 100, 250, 700])
def test_half_adder_records_bit_exact(kit, n):
    """Level widths 1..700 cover the cluster, latency, 2-per-CTA and 4-per-CTA
    kernels (and the narrow key-switch splits); AND / XOR outputs equal the
    oracle word for word and decrypt to the literals' AND / XOR."""
    engine, keys, octx = kit
    rng = np.random.default_rng(1000 + n)
    n_in = 64
    bits = rng.integers(0, 2, n_in).astype(np.uint8)
    cts = keys.encrypt(bits, seed=31, stream=n)
    recs = _ha_records(rng, n, n_in, n_in)
    engine.reserve(n_in + 2 * n)
    engine.upload(0, cts)
    engine.run_gates(recs)
    got = engine.download(n_in, 2 * n)
    pool = np.zeros((n_in + 2 * n, P.n + 1), np.uint32)
    pool[:n_in] = cts
    octx.run_gates(recs, pool, threads=os.cpu_count() or 1)
    assert np.array_equal(got, pool[n_in:])
    la = np.where(recs["alpha"] > 0, bits[recs["src_a"]], 1 - bits[recs["src_a"]])
    lb = np.where(recs["beta"] > 0, bits[recs["src_b"]], 1 - bits[recs["src_b"]])
    dec = keys.decrypt(got)
    assert np.array_equal(dec[:n], la & lb)
    # gamma = alpha * beta orients the second output to XOR of the underlying bits
    assert np.array_equal(dec[n:], bits[recs["src_a"]] ^ bits[recs["src_b"]])


def test_half_adder_with_lanes_and_mixed_level(engine, keys, octx):
    """HA records beside LIN2 / MUX / LIN3 records in one level, 3 lanes."""
    rng = np.random.default_rng(5)
    lanes, n_in, n_ha = 3, 40, 30
    bits = rng.integers(0, 2, (n_in, lanes)).astype(np.uint8)
    cts = keys.encrypt(bits.reshape(-1), seed=8, stream=3)
    ha = _ha_records(rng, n_ha, n_in, n_in)
    other = tfhe.gate_records(20)
    other["dst"] = n_in + 2 * n_ha + np.arange(20)
    srcs = rng.integers(0, n_in, (20, 3))
    other["src_a"], other["src_b"], other["src_c"] = srcs[:, 0], srcs[:, 1], srcs[:, 2]
    other["kind"] = np.arange(20) % 3
    c0, al, be = tfhe.GATE_LIN["XOR"]
    other["c0"] = np.where(other["kind"] == 0, c0, 0)
    other["alpha"] = np.where(other["kind"] == 0, al, 1)
    other["beta"] = np.where(other["kind"] == 0, be, -1)
    other["gamma"] = np.where(other["kind"] == 2, 1, 0)
    recs = np.concatenate([ha, other])
    rng.shuffle(recs)
    total = n_in + 2 * n_ha + 20
    engine.reserve(total * lanes)
    engine.upload(0, cts)
    engine.run_gates(recs, lanes=lanes)
    got = engine.download(n_in * lanes, (total - n_in) * lanes)
    exp = np.repeat(recs, lanes)
    lane = np.tile(np.arange(lanes, dtype=np.uint32), recs.size)
    for f in ("dst", "src_a", "src_b", "src_c"):
        exp[f] = exp[f] * lanes + lane
    pool = np.zeros((total * lanes, P.n + 1), np.uint32)
    pool[:n_in * lanes] = cts
    octx.run_gates(exp, pool, threads=os.cpu_count() or 1)
    assert np.array_equal(got, pool[n_in * lanes:])


def test_half_adder_phase_noise(engine, keys):
    """The XOR output carries two extractions' blind-rotation noise and one
    key switch: sigma^2 = 2 sigma_BR^2 + sigma_KS^2 (scripts/noise_budget.py);
    the measured phase error of 4,096 outputs stays within +-30% of it and far
    inside the 1/8 decryption margin."""
    rng = np.random.default_rng(77)
    n_in, n = 256, 4096
    bits = rng.integers(0, 2, n_in).astype(np.uint8)
    cts = keys.encrypt(bits, seed=12, stream=9)
    recs = _ha_records(rng, n, n_in, n_in)
    engine.reserve(n_in + 2 * n)
    engine.upload(0, cts)
    engine.run_gates(recs)
    got = engine.download(n_in, 2 * n)
    ph = keys.phase(got).astype(np.int64)
    la = np.where(recs["alpha"] > 0, bits[recs["src_a"]], 1 - bits[recs["src_a"]])
    lb = np.where(recs["beta"] > 0, bits[recs["src_b"]], 1 - bits[recs["src_b"]])
    want_bits = np.concatenate([la & lb, bits[recs["src_a"]] ^ bits[recs["src_b"]]])
    want = np.where(want_bits == 1, EIGHTH, -EIGHTH)
    err = ((ph - want + (1 << 31)) % (1 << 32) - (1 << 31)) / 2.0 ** 32
    s_and, s_xor = err[:n].std(), err[n:].std()
    s_br, s_ks = 2.0 ** -8.06, 2.0 ** -8.50  # DESIGN.md section 2 (key pairs)
    pred_and, pred_xor = np.hypot(s_br, s_ks), np.sqrt(2 * s_br ** 2 + s_ks ** 2)
    assert abs(s_and / pred_and - 1) < 0.3, (s_and, pred_and)
    assert abs(s_xor / pred_xor - 1) < 0.3, (s_xor, pred_xor)
    assert np.abs(err).max() < 0.125 / 2


def test_half_adder_level_split_into_chunks_is_identical():
    """A level of HA records (plus LIN2) wider than the per-launch work limit
    is split into chunks; each chunk numbers its second-extraction rows and
    XOR key switches locally, so the result must not depend on the split."""
    import subprocess
    import sys

    code = r'''
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_1806_03461_b200 import tfhe
keys = tfhe.KeySet(seed=42)
eng = tfhe.Engine(keys)
n, n_in = 300, 64
rng = np.random.default_rng(9)
eng.reserve(n_in + 2 * n)
eng.upload(0, keys.encrypt(rng.integers(0, 2, n_in).astype(np.uint8), seed=6, stream=1))
recs = tfhe.gate_records(n)
src = np.stack([rng.choice(n_in, 2, replace=False) for _ in range(n)])
recs["src_a"], recs["src_b"] = src[:, 0], src[:, 1]
recs["alpha"], recs["beta"] = rng.choice((-1, 1), n), rng.choice((-1, 1), n)
recs["gamma"] = recs["alpha"] * recs["beta"]
recs["c0"] = (-(1 << 29)) & 0xFFFFFFFF
recs["kind"] = np.where(np.arange(n) % 4 == 0, 0, 3)   # every 4th record a plain AND
recs["gamma"][recs["kind"] == 0] = 0
recs["dst"], recs["src_c"] = n_in + np.arange(n), n_in + n + np.arange(n)
eng.run_gates(recs)
np.save(sys.argv[1], eng.download(n_in, 2 * n))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for mw in ("0", "50"):
        path = f"/tmp/hb_ha_chunk_{mw}.npy"
        env = dict(os.environ)
        if mw != "0":
            env["HEBNN_B200_MAX_WORK"] = mw
        subprocess.run([sys.executable, "-c", code, path], check=True, cwd=root, env=env)
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])
