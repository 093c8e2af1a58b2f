"""The fast CPU baseline (oracle/tfhe_cpu_fft.c: FP64 FFT, eight gates per
SIMD register) against the exact-integer oracle: identical ciphertexts for
LIN2 / LIN3 gates, ragged block sizes, any thread count.  Test infrastructure
checking test infrastructure: bench.py times this port as `cpu_baseline` and
`--impl reference`, so its outputs must be the oracle's."""

import numpy as np
import pytest

from oracle import oracle as O

REC = np.dtype([("dst", "<u4"), ("src_a", "<u4"), ("src_b", "<u4"), ("src_c", "<u4"), ("c0", "<u4"),
                ("alpha", "i1"), ("beta", "i1"), ("kind", "i1"), ("gamma", "i1")])


@pytest.fixture(scope="module")
def setup():
    p = O.default_params()
    keys = O.Keys(p, 11)
    return p, keys, O.Context(p, keys), O.FftContext(p, keys)


def _pool(p, keys, gates, seed):
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2, (3, gates)).astype(np.uint8)
    pool = np.zeros((4 * gates, p.n + 1), np.uint32)
    for s in range(3):
        pool[s * gates:(s + 1) * gates] = O.encrypt(p, keys, bits[s], seed, s + 1)
    return bits, pool


@pytest.mark.parametrize("gates,threads", [(1, 1), (11, 3)])
def test_fft_port_is_bit_exact_vs_integer_oracle(setup, gates, threads):
    p, keys, exact, fft = setup
    bits, pool = _pool(p, keys, gates, 5 + gates)
    recs = np.zeros(gates, REC)
    names = list(O.GATE_LIN)
    for i in range(gates):
        if i % 4 == 3:  # LIN3: majority / XOR3
            c0, co = (0, 1) if i % 8 == 3 else (0, -2)
            recs[i] = (3 * gates + i, i, gates + i, 2 * gates + i, c0, co, co, 2, co)
        else:
            c0, al, be = O.GATE_LIN[names[i % len(names)]]
            recs[i] = (3 * gates + i, i, gates + i, 0, c0, al, be, 0, 0)
    p_exact, p_fft = pool.copy(), pool.copy()
    exact.run_gates(recs, p_exact, threads=threads)
    fft.run_gates(recs, p_fft, threads=threads)
    assert np.array_equal(p_exact, p_fft)
    out = O.decrypt(p, keys, p_fft[3 * gates:])
    for i in range(gates):
        a, b, c = int(bits[0, i]), int(bits[1, i]), int(bits[2, i])
        if i % 4 == 3:
            want = int(a + b + c >= 2) if i % 8 == 3 else (a ^ b ^ c)
        else:
            want = {"AND": a & b, "OR": a | b, "XOR": a ^ b, "XNOR": 1 - (a ^ b), "NAND": 1 - (a & b),
                    "NOR": 1 - (a | b)}[names[i % len(names)]]
        assert out[i] == want


def test_fft_port_rejects_other_kinds_and_layouts(setup):
    p, keys, _, fft = setup
    _, pool = _pool(p, keys, 1, 3)
    recs = np.zeros(1, REC)
    recs[0] = (3, 0, 1, 2, 0, 1, 1, 1, 0)  # MUX
    with pytest.raises(ValueError):
        fft.run_gates(recs, pool)
    q = O.default_params()
    q.bk_unroll = 1
    with pytest.raises(ValueError):
        O.FftContext(q, O.Keys(q, 3))
