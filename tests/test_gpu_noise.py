"""Phase-noise monitor: bootstrapped outputs carry the noise the parameter set
predicts (scripts/noise_budget.py: fresh gate output sigma = 2^-8.15 of the
torus with the CGGI key, 2^-7.75 with the key-pair key), far inside the 1/8
decryption margin."""

import math

import numpy as np
import pytest

from paper_1806_03461_b200 import tfhe

pytestmark = pytest.mark.gpu
SIGMA_OUT = {1: 2.0 ** -8.15, 2: 2.0 ** -7.75}  # scripts/noise_budget.py


@pytest.mark.parametrize("unroll", [2, 1])
def test_gate_output_noise_matches_budget(unroll):
    p = tfhe.default_params()
    p.bk_unroll = unroll
    keys = tfhe.KeySet(seed=5, params=p)
    eng = tfhe.Engine(keys)
    n = 2048
    rng = np.random.default_rng(2)
    a = rng.integers(0, 2, n).astype(np.uint8)
    b = rng.integers(0, 2, n).astype(np.uint8)
    eng.reserve(3 * n)
    eng.upload(0, keys.encrypt(a, seed=5, stream=1))
    eng.upload(n, keys.encrypt(b, seed=5, stream=2))
    for name in ("NAND", "XOR"):
        c0, al, be = tfhe.GATE_LIN[name]
        recs = tfhe.gate_records(n)
        recs["dst"], recs["src_a"], recs["src_b"] = np.arange(2 * n, 3 * n), np.arange(n), np.arange(n, 2 * n)
        recs["c0"], recs["alpha"], recs["beta"] = c0, al, be
        eng.run_gates(recs)
        out = eng.download(2 * n, n)
        want = (1 - (a & b)) if name == "NAND" else (a ^ b)
        assert np.array_equal(keys.decrypt(out), want)
        ph = keys.phase(out).astype(np.int64)
        noise = (ph - np.where(want == 1, 1 << 29, -(1 << 29))) / 2.0 ** 32
        sigma = float(noise.std())
        assert 0.7 * SIGMA_OUT[unroll] < sigma < 1.3 * SIGMA_OUT[unroll], (name, math.log2(sigma))
        assert float(np.abs(noise).max()) < 1.0 / 16  # half the decryption margin
    eng.close()
