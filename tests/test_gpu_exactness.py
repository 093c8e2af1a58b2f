"""The FP64-FFT exactness claim as a tested bound.

The blind rotation computes every negacyclic product in FP64 and rounds it
back to the 2^32 torus; it is bit-exact with the integer oracle only while
every inverse-FFT output lies within 0.5 of its integer.  Per key layout:

* >= 16,384 bootstraps through the instrumented (kDebug) kernels: half
  uniformly random LWE samples (arbitrary rotations, a pseudo-random
  accumulator after a few steps), half structured extremes (all-max / all-zero
  / half-turn masks, bodies on the phase boundaries 0, +-1/8, +-1/4, 1/2, and
  constant accumulators whose digit polynomials are maximal and constant)
  -> max |x - round(x)| < 0.1 (a 5x safety factor below the exactness bound);
* a sample of those bootstraps bit-exact against the exact-integer oracle;
* the production kernels (run_gates) on 16,384 gates, three times: identical
  output words every time (no race in the exchange / ring barriers), and a
  sample bit-exact against the oracle's gate.

Reference contract: /root/reference/pkg/src/hebnn/backend.py:188-190 (decrypt
returns the simulated bit); bit-exact ciphertexts are checked against our own
exact-integer restatement (oracle/tfhe_oracle.c), the reference having none.
"""

import numpy as np
import pytest

from paper_1806_03461_b200 import tfhe

pytestmark = pytest.mark.gpu

COUNT = 16384
MARGIN_BOUND = 0.1


@pytest.fixture(params=["pairs", "cggi"])
def kit(request):
    sfx = "" if request.param == "pairs" else "1"
    return tuple(request.getfixturevalue(name + sfx) for name in ("engine", "keys", "octx"))


def _stress_inputs(keys, count, seed):
    """count LWE samples [count][n+1]: half uniform, half structured extremes."""
    n = keys.params.n
    rng = np.random.default_rng(seed)
    half = count // 2
    lin = np.zeros((count, n + 1), np.uint32)
    lin[:half] = rng.integers(0, 2 ** 32, (half, n + 1), dtype=np.uint64).astype(np.uint32)
    bodies = np.array([0, 1 << 29, (-(1 << 29)) & 0xFFFFFFFF, 1 << 30, (-(1 << 30)) & 0xFFFFFFFF, 1 << 31,
                       (1 << 29) - 1, (1 << 29) + 1, 0xFFFFFFFF, 1], dtype=np.uint32)
    masks = [
        lambda k: np.zeros((k, n), np.uint32),                           # no rotation: constant accumulator
        lambda k: np.full((k, n), 0xFFFFFFFF, np.uint32),                # all-max
        lambda k: np.full((k, n), 1 << 31, np.uint32),                   # half turns (X^N = -1)
        lambda k: np.full((k, n), 1 << 21, np.uint32),                   # one-step rotations
        lambda k: rng.choice(np.array([0, 1 << 31, 0xFFFFFFFF, 1 << 21], np.uint32), (k, n)),
        lambda k: (rng.integers(0, 2048, (k, n)) << 21).astype(np.uint32),  # exact mod-switch grid
    ]
    rows = np.array_split(np.arange(half, count), len(masks))
    for mk, idx in zip(masks, rows):
        lin[idx, :n] = mk(idx.size)
        lin[idx, n] = bodies[rng.integers(0, bodies.size, idx.size)]
    return lin


def test_fft_rounding_margin_and_oracle_sample(kit):
    engine, keys, octx = kit
    lin = _stress_inputs(keys, COUNT, seed=2024 + keys.params.bk_unroll)
    worst = 0.0
    outs = []
    for part in np.array_split(np.arange(COUNT), 4):
        outs.append(engine.debug_bootstrap_wo_ks(lin[part]))
        worst = max(worst, engine.debug_fft_margin())
    got = np.concatenate(outs)
    assert worst < MARGIN_BOUND, f"FFT rounding margin {worst} (bk_unroll={keys.params.bk_unroll})"
    rng = np.random.default_rng(5)
    sample = np.concatenate([rng.choice(COUNT // 2, 6, replace=False),
                             COUNT // 2 + rng.choice(COUNT // 2, 10, replace=False)])
    for i in sample:
        assert np.array_equal(got[i], octx.bootstrap_wo_ks(lin[i])), int(i)
    # the instrumented kernel is deterministic too
    again = engine.debug_bootstrap_wo_ks(lin[:2048])
    assert np.array_equal(again, got[:2048])


def test_production_kernels_deterministic_and_exact(kit):
    engine, keys, octx = kit
    rng = np.random.default_rng(77 + keys.params.bk_unroll)
    n = COUNT
    a = rng.integers(0, 2, n).astype(np.uint8)
    b = rng.integers(0, 2, n).astype(np.uint8)
    ca, cb = keys.encrypt(a, seed=61, stream=1), keys.encrypt(b, seed=61, stream=2)
    engine.reserve(3 * n)
    engine.upload(0, ca)
    engine.upload(n, cb)
    recs = tfhe.gate_records(n)
    # a mix of gate kinds exercises every prologue sign combination
    kinds = list(tfhe.GATE_LIN)
    pick = rng.integers(0, len(kinds), n)
    for k, name in enumerate(kinds):
        c0, al, be = tfhe.GATE_LIN[name]
        sel = pick == k
        recs["c0"][sel], recs["alpha"][sel], recs["beta"][sel] = c0, al, be
    recs["dst"], recs["src_a"], recs["src_b"] = 2 * n + np.arange(n), np.arange(n), n + np.arange(n)
    runs = []
    for _ in range(3):
        engine.run_gates(recs)
        runs.append(engine.download(2 * n, n))
    assert np.array_equal(runs[0], runs[1]) and np.array_equal(runs[0], runs[2])
    for i in rng.choice(n, 8, replace=False):
        want = octx.gate(int(recs["c0"][i]), int(recs["alpha"][i]), ca[i], int(recs["beta"][i]), cb[i])
        assert np.array_equal(runs[0][i], want), int(i)
