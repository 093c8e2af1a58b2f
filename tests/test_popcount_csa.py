"""Carry-save popcount (paper_1806_03461_b200/popcount.py, Dag.csa): same words,
same counted stats as the reference's reduce_tree_sum (circuits.py:189-216),
fewer executed bootstraps.  CPU: host logic on the plaintext stand-in engine."""

import math
import random

import pytest

import hebnn.circuits as ref_circuits
from hebnn.backend import SimContext
from hebnn.circuits import decrypt_word
from hebnn.compiler import EvalOptions, decrypt_output, encrypt_input, eval_model
from hebnn.model import DenseLayer, SignActivation, TernaryModel, oracle_eval, validate_model

from paper_1806_03461_b200 import popcount
from plain_engine import plain_context_class

Plain = plain_context_class()


@pytest.fixture(autouse=True)
def _restore_reference_binding():
    yield
    popcount.uninstall()


def _sum_word(ctx, bits):
    return ref_circuits.reduce_tree_sum([ctx.encrypt(b) for b in bits])


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 31, 33, 63, 64, 100, 255, 256, 257, 392, 784])
def test_popcount_words_and_stats_match_the_reference(n):
    rng = random.Random(n)
    for trial in range(3):
        bits = [1] * n if trial == 0 else ([0] * n if trial == 1 else [rng.randint(0, 1) for _ in range(n)])
        sim = SimContext()
        want = _sum_word(sim, bits)
        ctx = Plain(seed=42, csa_popcount=True)
        got = _sum_word(ctx, bits)
        assert got.width == want.width == max(1, math.ceil(math.log2(n + 1)))
        assert got.max_value == want.max_value and got.signed == want.signed
        assert [b.level for b in got.bits] == [b.level for b in want.bits]
        assert decrypt_word(got) == decrypt_word(want) == sum(bits)
        assert ctx.global_stats.as_dict() == sim.global_stats.as_dict()


def test_fewer_bootstraps_than_the_ripple_tree():
    n = 392
    bits = [random.Random(1).randint(0, 1) for _ in range(n)]
    base = Plain(seed=42)
    assert decrypt_word(_sum_word(base, bits)) == sum(bits)
    ctx = Plain(seed=42, csa_popcount=True)
    assert decrypt_word(_sum_word(ctx, bits)) == sum(bits)
    assert ctx.gate_count == base.gate_count
    # full adders cost two bootstraps: ~2n against ~3n
    assert ctx.exec_stats["bootstraps"] <= 2 * n
    assert ctx.exec_stats["bootstraps"] < 0.75 * base.exec_stats["bootstraps"]


def test_negated_and_mixed_level_bits_and_scopes():
    rng = random.Random(5)
    vals = [rng.randint(0, 1) for _ in range(40)]

    def run(ctx):
        xs = [ctx.encrypt(v) for v in vals]
        deep = [ctx.g_and(xs[i], xs[i + 1]) for i in range(0, 20, 2)]       # level-1 bits
        lits = [ctx.g_not(x) for x in xs[20:30]] + xs[30:] + deep             # negated, plain, deeper
        ctx.begin_scope("sum")
        word = ref_circuits.reduce_tree_sum(lits)
        scope = ctx.end_scope()
        return decrypt_word(word), [b.level for b in word.bits], scope.as_dict(), ctx.global_stats.as_dict()

    assert run(Plain(seed=42, csa_popcount=True)) == run(SimContext())


def test_other_contexts_and_trivial_bits_use_the_reference_circuit():
    Plain(seed=42, csa_popcount=True)  # installs the rebinding
    assert popcount.installed()
    sim = SimContext()
    assert decrypt_word(_sum_word(sim, [1, 1, 0, 1, 1])) == 4
    pure = Plain(seed=42)
    base = Plain(seed=42)
    popcount.uninstall()
    w0 = _sum_word(base, [1, 1, 0, 1, 1, 0, 1])
    popcount.install()
    w1 = _sum_word(pure, [1, 1, 0, 1, 1, 0, 1])
    assert decrypt_word(w0) == decrypt_word(w1) == 5
    assert pure.exec_stats["bootstraps"] == base.exec_stats["bootstraps"]
    ctx = Plain(seed=42, csa_popcount=True)
    word = ref_circuits.reduce_tree_sum([ctx.encrypt(1), ctx.trivial_const(1), ctx.encrypt(1), ctx.encrypt(0)])
    assert decrypt_word(word) == 3
    x = ctx.encrypt(1)
    assert decrypt_word(ref_circuits.reduce_tree_sum([x, x, ctx.g_not(x), ctx.encrypt(1)])) == 3


def test_models_match_oracle_eval_and_simcontext_stats():
    rng = random.Random(11)
    for trial in range(6):
        d, p = rng.randint(8, 60), rng.randint(1, 4)
        rows = tuple(tuple(rng.choice((-1, 0, 1) if trial % 2 else (-1, 1)) for _ in range(d)) for _ in range(p))
        mode = "score_words" if trial % 3 == 0 else "sign_bits"
        layers = (DenseLayer(rows, tuple(rng.randint(-3, 3) for _ in range(p))),)
        if mode == "sign_bits":
            layers += (SignActivation(),)
        m = validate_model(TernaryModel(d, layers, mode))
        xs = [rng.choice((-1, 1)) for _ in range(d)]
        for opts in (EvalOptions(), EvalOptions(plus_one=False), EvalOptions(comparator="sort")):
            sim = SimContext()
            eval_model(sim, m, encrypt_input(sim, xs), opts)
            base = Plain(seed=42)
            popcount.uninstall()
            outs, _ = eval_model(base, m, encrypt_input(base, xs), opts)
            assert decrypt_output(base, outs) == oracle_eval(m, xs)
            c = Plain(seed=42, csa_popcount=True)
            outs, _ = eval_model(c, m, encrypt_input(c, xs), opts)
            assert decrypt_output(c, outs) == oracle_eval(m, xs)
            assert c.global_stats.as_dict() == sim.global_stats.as_dict()
            assert c.exec_stats["bootstraps"] <= base.exec_stats["bootstraps"]


@pytest.mark.parametrize("block", [0, 3, 5, 7, 12])
def test_shared_first_stage_block_sizes(block, monkeypatch):
    """Any block size of the shared first stage (HEBNN_B200_CSA_BLOCK; 0: none) gives the
    same words; popcounts over subsets of one input vector reuse each other's adders."""
    monkeypatch.setenv("HEBNN_B200_CSA_BLOCK", str(block))
    rng = random.Random(block)
    vals = [rng.randint(0, 1) for _ in range(120)]
    ctx = Plain(seed=42, csa_popcount=True)
    assert ctx.csa_block == block
    xs = [ctx.encrypt(v) for v in vals]
    subsets = [[i for i in range(120) if rng.random() < 0.5] for _ in range(12)]
    words = [ref_circuits.reduce_tree_sum([xs[i] if k % 2 else ctx.g_not(xs[i]) for i in sub])
             for k, sub in enumerate(subsets)]
    for k, (sub, w) in enumerate(zip(subsets, words)):
        assert decrypt_word(w) == sum(vals[i] if k % 2 else 1 - vals[i] for i in sub)
    total_bits = sum(len(sub) for sub in subsets)
    assert ctx.exec_stats["bootstraps"] < 2 * total_bits
    if block >= 3:  # shared adders: clearly fewer than twelve independent networks
        assert ctx.exec_stats["bootstraps"] < 1.9 * total_bits


def test_environment_default(monkeypatch):
    monkeypatch.setenv("HEBNN_B200_CSA_POPCOUNT", "1")
    assert Plain(seed=42).csa_popcount is True
    assert Plain(seed=42, csa_popcount=False).csa_popcount is False
    monkeypatch.setenv("HEBNN_B200_CSA_POPCOUNT", "0")
    assert Plain(seed=42).csa_popcount is False


def test_duplicate_and_complementary_literals_property():
    """Random multisets of literals with repeated and complementary bits (the degenerate
    operands of Dag.csa: XOR / MAJ / AND folding to constants or single literals): the word
    is the number of true literals whatever path (compressor network or the fallback to the
    reference circuit when a digit folds to a constant) built it."""
    rng = random.Random(77)
    for trial in range(60):
        ctx = Plain(seed=42, csa_popcount=True, stream_at=0)
        k = rng.randint(1, 6)
        vals = [rng.randint(0, 1) for _ in range(k)]
        xs = [ctx.encrypt(v) for v in vals]
        n = rng.randint(3, 40)
        picks = [(rng.randrange(k), rng.randint(0, 1)) for _ in range(n)]
        lits = [ctx.g_not(xs[i]) if neg else xs[i] for i, neg in picks]
        sim = SimContext()
        sx = [sim.encrypt(v) for v in vals]
        want_word = ref_circuits.reduce_tree_sum([sim.g_not(sx[i]) if neg else sx[i] for i, neg in picks])
        word = ref_circuits.reduce_tree_sum(lits)
        want = sum(1 - vals[i] if neg else vals[i] for i, neg in picks)
        assert decrypt_word(word) == decrypt_word(want_word) == want, (trial, picks)
        assert word.width == want_word.width
        assert ctx.global_stats.as_dict() == sim.global_stats.as_dict()
