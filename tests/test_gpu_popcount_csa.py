"""Carry-save popcount (TfheContext(csa_popcount=True), popcount.py) on real
CGGI ciphertexts: the compiler's popcounts run as Wallace-style compressor
networks built by Dag.csa.  Decrypted outputs equal the reference's
oracle_eval (model.py:458-497), counted stats equal SimContext's
(backend.py:161-257), executed bootstraps drop by about 40%."""

import random

import numpy as np
import pytest

import hebnn.circuits as ref_circuits
from hebnn.backend import SimContext
from hebnn.circuits import compare_ge_const, decrypt_word
from hebnn.compiler import EvalOptions, decrypt_output, encrypt_input, eval_model
from hebnn.model import DenseLayer, SignActivation, TernaryModel, oracle_eval, validate_model
from paper_1806_03461_b200 import popcount
from paper_1806_03461_b200.backend import TfheContext

pytestmark = pytest.mark.gpu


class CsaContext(TfheContext):
    def __init__(self, **kw):
        kw.setdefault("csa_popcount", True)
        super().__init__(**kw)


@pytest.fixture(autouse=True)
def _restore_reference_binding():
    yield
    popcount.uninstall()


# the reference's reduce-tree tests (test_circuits.py:109-141) on the compressor network
@pytest.mark.parametrize("n", [3, 4, 7, 12, 33, 100, 392])
def test_popcount_words_on_gpu(n):
    rng = random.Random(n)
    ctx, sim = CsaContext(seed=42), SimContext()
    cases = [[1] * n, [0] * n] + [[rng.randint(0, 1) for _ in range(n)] for _ in range(3)]
    words = [ref_circuits.reduce_tree_sum([ctx.encrypt(b) for b in bits]) for bits in cases]
    ges = [compare_ge_const(w, (n + 1) // 2) for w in words]
    for bits in cases:
        compare_ge_const(ref_circuits.reduce_tree_sum([sim.encrypt(b) for b in bits]), (n + 1) // 2)
    for bits, w, g in zip(cases, words, ges):
        assert decrypt_word(w) == sum(bits)
        assert ctx.decrypt(g) == int(sum(bits) >= (n + 1) // 2)
    assert ctx.global_stats.as_dict() == sim.global_stats.as_dict()
    assert ctx.exec_stats["bootstraps"] < ctx.gate_count


def test_exhaustive_small_popcounts_in_lanes():
    """Every input pattern of n = 5 and n = 9 bits (test_circuits.py:124-130), one lane per pattern."""
    for n in (5, 9):
        pats = np.array([[(p >> i) & 1 for p in range(1 << n)] for i in range(n)], np.uint8)  # [n][2^n]
        ctx = CsaContext(seed=42, lanes=1 << n)
        word = ref_circuits.reduce_tree_sum([ctx.encrypt_lanes(pats[i]) for i in range(n)])
        got = sum(np.asarray(ctx.decrypt(b)).astype(np.int64) << i for i, b in enumerate(word.bits))
        assert np.array_equal(got, pats.sum(axis=0))


def test_random_models_match_oracle_eval_and_simcontext_stats():
    rng = random.Random(21)
    for trial in range(8):
        d, p = rng.randint(8, 96), rng.randint(1, 5)
        rows = tuple(tuple(rng.choice((-1, 0, 1) if trial % 2 else (-1, 1)) for _ in range(d)) for _ in range(p))
        mode = "score_words" if trial % 3 == 0 else "sign_bits"
        layers = (DenseLayer(rows, tuple(rng.randint(-3, 3) for _ in range(p))),)
        if mode == "sign_bits":
            layers += (SignActivation(),)
        m = validate_model(TernaryModel(d, layers, mode))
        xs = [rng.choice((-1, 1)) for _ in range(d)]
        opts = (EvalOptions(), EvalOptions(plus_one=False), EvalOptions(comparator="sort"))[trial % 3]
        sim = SimContext()
        eval_model(sim, m, encrypt_input(sim, xs), opts)
        ctx = CsaContext(seed=42)
        outs, _ = eval_model(ctx, m, encrypt_input(ctx, xs), opts)
        assert decrypt_output(ctx, outs) == oracle_eval(m, xs)
        assert ctx.global_stats.as_dict() == sim.global_stats.as_dict()


@pytest.mark.parametrize("config", ["cfg2n", "cfg2l", "cfg3", "cfg4", "cfg5", "conv"])
def test_baseline_configs_full_size_with_csa_popcount(config, tmp_path):
    """Every BASELINE.json BNN config at full size with the carry-save popcount:
    first evaluation, a replay on a second encrypted batch and a fresh context
    running the compiled schedule all equal oracle_eval; counted gates and depth
    are SimContext's; the executed bootstraps are well below the drop-in's
    (~0.30 of the counted gates instead of ~0.33-0.45)."""
    from paper_1806_03461_b200 import workloads

    big = config in ("cfg3", "cfg5")
    rep = workloads.run_encrypted(CsaContext, config, seed=0, replays=0 if big else 1, cached=not big,
                                  schedule_path=None if big else str(tmp_path / f"{config}.sched.npz"))
    assert rep["matches_oracle_eval"] is True
    if not big:
        assert rep["replay"]["matches_oracle_eval"] is True
        assert rep["cached"]["matches_oracle_eval"] is True
    popcount.uninstall()
    sim = workloads.run_sim_reference(config, seed=0)
    assert rep["counted_gates_per_input"] == sim["counted_gates_per_input"]
    assert rep["executed_bootstraps"] < 0.30 * rep["counted_gates"]


def test_cancer_rows_with_csa_popcount():
    from paper_1806_03461_b200 import workloads

    rep = workloads.run_cancer(CsaContext, seed=0)
    assert rep["matches_oracle_eval"] is True
    assert abs(rep["accuracy_test"] - rep["trainer_accuracy"]["test"]) < 1e-12
