"""CPU oracle checks (no GPU): exact negacyclic products, keygen/encryption
parity between the oracle restatement and the product's host code, and the
oracle against the committed golden vectors (tests/golden/)."""

import os

import numpy as np
import pytest

from oracle import oracle as O

P = O.default_params()
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "tfhe_golden_seed42.npz")
GOLDEN_PAIRS = os.path.join(os.path.dirname(__file__), "golden", "tfhe_golden_pairs_seed42.npz")


def test_default_params_match_baseline():
    # BASELINE.json configs[0]
    assert (P.n, P.N, P.k, P.bg_bits, P.l, P.ks_base_bits, P.ks_t) == (630, 1024, 1, 7, 3, 2, 8)
    assert P.lwe_stdev == 2.0 ** -15 and P.bk_stdev == 2.0 ** -25
    assert P.bk_unroll == 2  # key-pair bootstrapping key by default; 1 = one TGSW per key bit


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_ntt_product_equals_schoolbook_mod_2_32(seed):
    rng = np.random.default_rng(seed)
    a = rng.integers(-64, 64, 1024).astype(np.int32)  # gadget digits
    b = rng.integers(0, 2 ** 32, 1024, dtype=np.uint64).astype(np.uint32)
    assert np.array_equal(O.negacyclic_mul(a, b, "ntt"), O.negacyclic_mul(a, b, "school"))


def test_negacyclic_identity_monomials():
    # X^i * X^(N-i) = X^N = -1
    a = np.zeros(1024, np.int32)
    a[3] = 1
    b = np.zeros(1024, np.uint32)
    b[1021] = 5
    out = O.negacyclic_mul(a, b)
    want = np.zeros(1024, np.uint32)
    want[0] = (-5) & 0xFFFFFFFF
    assert np.array_equal(out, want)


def test_product_keygen_and_encrypt_bit_identical_to_oracle(keys, okeys):
    assert np.array_equal(keys.lwe_key, okeys.lwe_key)
    assert np.array_equal(keys.trlwe_key, okeys.trlwe_key)
    assert np.array_equal(keys.bk, okeys.bk.reshape(-1))
    assert np.array_equal(keys.ksk, okeys.ksk.reshape(-1))
    bits = np.random.default_rng(3).integers(0, 2, 64).astype(np.uint8)
    for stream, first in ((0, 0), (7, 1000)):
        mine = keys.encrypt(bits, seed=5, stream=stream, first_index=first)
        theirs = O.encrypt(P, okeys, bits, 5, stream, first)
        assert np.array_equal(mine, theirs)


def test_encrypt_decrypt_roundtrip_and_noise(okeys):
    bits = np.random.default_rng(4).integers(0, 2, 1000).astype(np.uint8)
    cts = O.encrypt(P, okeys, bits, 9, 1)
    assert np.array_equal(O.decrypt(P, okeys, cts), bits)
    ph = O.phase(P, okeys, cts).astype(np.int64)
    err = ph - np.where(bits == 1, 1 << 29, -(1 << 29))
    # fresh noise: sigma = 2^-15 * 2^32 = 2^17
    assert np.abs(err).max() < 8 * (1 << 17)


def test_encrypt_rejects_non_bits(okeys):
    with pytest.raises(ValueError):
        O.encrypt(P, okeys, np.array([2], np.uint8), 1, 1)


def test_keyswitch_key_decrypts_to_scaled_key_bits(okeys):
    # KSK[i][j][v-1] encrypts v * s'_i / 4^(j+1) under the LWE key
    for i, j, v in ((0, 0, 1), (5, 3, 2), (1023, 7, 3)):
        ct = okeys.ksk[i, j, v - 1]
        ph = int(O.phase(P, okeys, ct)[0]) & 0xFFFFFFFF
        msg = (int(okeys.trlwe_key[i]) * v << (32 - 2 * (j + 1))) & 0xFFFFFFFF
        diff = (ph - msg + 2 ** 31) % 2 ** 32 - 2 ** 31
        assert abs(diff) < 8 * (1 << 17)


@pytest.mark.skipif(not os.path.exists(GOLDEN), reason="golden vectors not generated")
def _check_golden(path, okeys, octx, prefix_iters):
    g = np.load(path)
    assert g["lwe_key"].tobytes() == okeys.lwe_key.tobytes()
    assert int(g["bk_sum"]) == int(okeys.bk.astype(np.uint64).sum())
    assert int(g["ksk_sum"]) == int(okeys.ksk.astype(np.uint64).sum())
    inputs = g["inputs"]
    assert np.array_equal(O.encrypt(P, okeys, g["input_bits"], 42, 77), inputs)
    assert np.array_equal(octx.blind_rotate(inputs[0], iters=prefix_iters), g["acc_prefix3"])
    assert np.array_equal(octx.keyswitch(g["ks_in"]), g["ks_out"])
    for name, (c0, al, be) in O.GATE_LIN.items():
        if name in ("AND", "XOR"):
            out = octx.gate(c0, al, inputs[0], be, inputs[1])
            assert np.array_equal(out, g[f"gate_{name}"]), name


def test_oracle_reproduces_golden_vectors(okeys1, octx1):
    """CGGI layout (bk_unroll 1)."""
    _check_golden(GOLDEN, okeys1, octx1, 3)


def test_oracle_reproduces_golden_vectors_key_pairs(okeys, octx):
    """Key-pair layout (bk_unroll 2, the default)."""
    _check_golden(GOLDEN_PAIRS, okeys, octx, 4)


def test_cggi_key_layout_bit_identical_to_oracle(keys1, okeys1):
    assert np.array_equal(keys1.bk, okeys1.bk.reshape(-1))
    assert np.array_equal(keys1.ksk, okeys1.ksk.reshape(-1))


def _acc_phase(okeys, acc):
    """Phase polynomial B - A*s of a TRLWE accumulator (exact)."""
    A, B = acc[:1024], acc[1024:]
    s = okeys.trlwe_key.astype(np.int32)
    return (B - O.negacyclic_mul(s, A)).astype(np.uint32).view(np.int32).astype(np.int64)


def test_key_pair_blind_rotation_equals_cggi_blind_rotation(okeys, octx, okeys1, octx1):
    """The key-pair CMux rotates the accumulator by X^{a_i s_i + a_j s_j} per
    pair, so after the whole key both layouts hold X^{sum a_i s_i - b} * TV:
    identical message polynomials (+-1/8 per coefficient), independent noise."""
    assert np.array_equal(okeys.lwe_key, okeys1.lwe_key)
    rng = np.random.default_rng(8)
    for trial in range(3):
        lwe = O.encrypt(P, okeys, rng.integers(0, 2, 1).astype(np.uint8), 3, 40 + trial)[0]
        ph2 = _acc_phase(okeys, octx.blind_rotate(lwe))
        ph1 = _acc_phase(okeys1, octx1.blind_rotate(lwe))
        eighth = 1 << 29
        for ph in (ph1, ph2):
            assert np.all(np.abs(np.abs(ph) - eighth) < eighth // 4)
        assert np.array_equal(np.sign(ph1), np.sign(ph2))
