"""The reference's decrypted-result tests restated on TfheContext, i.e. on
real CGGI ciphertexts bootstrapped by the sm_100a engine.  Each test names the
reference test it restates; circuits are built first and decrypted together
(one flush, one device batch per level) — the assertions are the reference's.
"""

import itertools
import json
import os
import random

import numpy as np
import pytest

from hebnn.backend import AND, MUX, OR, XNOR, XOR, SimContext
from hebnn.circuits import (
    compare_ge_const,
    compare_signed_ge_const,
    decrypt_word,
    encrypt_word,
    half_adder,
    rc_add,
    rc_sub,
    reduce_tree_sum,
)
from hebnn.compiler import EvalOptions, decrypt_output, encrypt_input, eval_model
from hebnn.model import (
    BatchNorm,
    ConvLayer,
    DenseLayer,
    SignActivation,
    TernaryModel,
    oracle_eval,
    validate_model,
)
from paper_1806_03461_b200.backend import TfheContext

pytestmark = pytest.mark.gpu
PLAIN = {AND: lambda a, b: a & b, OR: lambda a, b: a | b, XOR: lambda a, b: a ^ b, XNOR: lambda a, b: 1 - (a ^ b)}
HERE = os.path.dirname(os.path.abspath(__file__))


def ctx_new(**kw):
    return TfheContext(seed=42, **kw)


# test_backend.py:52-58
@pytest.mark.parametrize("kind", [AND, OR, XOR, XNOR])
def test_gate_truth_tables_exhaustive(kind):
    ctx = ctx_new()
    fn = {AND: ctx.g_and, OR: ctx.g_or, XOR: ctx.g_xor, XNOR: ctx.g_xnor}[kind]
    outs = [(a, b, fn(ctx.encrypt(a), ctx.encrypt(b))) for a in (0, 1) for b in (0, 1)]
    for a, b, o in outs:
        assert ctx.decrypt(o) == PLAIN[kind](a, b)


# test_backend.py:116-123
def test_mux_exhaustive():
    ctx = ctx_new()
    outs = [(s, a, b, ctx.g_mux(ctx.encrypt(s), ctx.encrypt(a), ctx.encrypt(b)))
            for s, a, b in itertools.product((0, 1), repeat=3)]
    for s, a, b, o in outs:
        assert ctx.decrypt(o) == (a if s else b)
    assert ctx.global_stats.counts[MUX] == 8


# test_backend.py:80-83, 97-106
def test_decrypt_trivial_gate_output_and_not():
    ctx = ctx_new()
    assert ctx.decrypt(ctx.trivial_const(1)) == 1
    assert ctx.decrypt(ctx.g_and(ctx.encrypt(1), ctx.encrypt(0))) == 0
    a = ctx.encrypt(1)
    for _ in range(50):
        a = ctx.g_not(a)
    assert ctx.decrypt(a) == 1 and ctx.decrypt(ctx.g_not(a)) == 0


# test_backend.py:200-213 (256 random sequences, one context, one flush)
def test_random_gate_sequences_match_plain_boolean_eval():
    rng = random.Random(123)
    ctx = ctx_new()
    checks = []
    for _ in range(256):
        values = [rng.randint(0, 1) for _ in range(4)]
        enc = [ctx.encrypt(v) for v in values]
        plain = list(values)
        for _ in range(rng.randint(1, 12)):
            kind = rng.choice([AND, OR, XOR, XNOR])
            i, j = rng.randrange(len(plain)), rng.randrange(len(plain))
            enc.append({AND: ctx.g_and, OR: ctx.g_or, XOR: ctx.g_xor, XNOR: ctx.g_xnor}[kind](enc[i], enc[j]))
            plain.append(PLAIN[kind](plain[i], plain[j]))
        checks.extend(zip(enc, plain))
    got = ctx.decrypt_many([e for e, _ in checks])[:, 0]
    assert [int(g) for g in got] == [p for _, p in checks]


# test_circuits.py:36-42, 60-68, 76-82
def test_adders_exhaustive_k4():
    ctx = ctx_new()
    has = [(a, b, half_adder(ctx.encrypt(a), ctx.encrypt(b))) for a, b in itertools.product((0, 1), repeat=2)]
    adds = [(x, y, rc_add(encrypt_word(ctx, x, 4), encrypt_word(ctx, y, 4))) for x, y in itertools.product(range(16), repeat=2)]
    subs = [(x, y, rc_sub(encrypt_word(ctx, x, 4), encrypt_word(ctx, y, 4))) for x, y in itertools.product(range(16), repeat=2)]
    ctx.flush()
    for a, b, (s, c) in has:
        assert (ctx.decrypt(s), ctx.decrypt(c)) == ((a + b) % 2, (a + b) // 2)
    for x, y, w in adds:
        assert decrypt_word(w) == x + y
    for x, y, w in subs:
        assert decrypt_word(w) == x - y


# test_circuits.py:124-130 (exhaustive reduce tree, n <= 8 here)
def test_reduce_tree_exhaustive_small_n():
    ctx = ctx_new()
    runs = []
    for n in range(1, 9):
        for mask in range(1 << n):
            bits = [(mask >> i) & 1 for i in range(n)]
            runs.append((sum(bits), reduce_tree_sum([ctx.encrypt(b) for b in bits])))
    ctx.flush()
    for want, word in runs:
        assert decrypt_word(word) == want


# test_circuits.py:216-223, 250-258 (comparators exhaustive, k=6 unsigned / k=5 signed)
def test_comparators_exhaustive():
    ctx = ctx_new()
    runs = []
    k = 6
    for value in range(1 << k):
        word = encrypt_word(ctx, value, k)
        for thr in range(-1, (1 << k) + 2):
            runs.append((int(value >= thr), compare_ge_const(word, thr)))
    k = 5
    lo, hi = -(1 << (k - 1)), (1 << (k - 1)) - 1
    for value in range(lo, hi + 1):
        word = encrypt_word(ctx, value, k, signed=True)
        for thr in range(lo - 1, hi + 2):
            runs.append((int(value >= thr), compare_signed_ge_const(word, thr)))
    ctx.flush()
    got = ctx.decrypt_many([h for _, h in runs])[:, 0]
    assert [int(g) for g in got] == [w for w, _ in runs]


# test_compiler.py:150-165 (neurons exhaustive over inputs, d <= 4)
@pytest.mark.parametrize("plus_one", [True, False])
def test_neurons_exhaustive_d4(plus_one):
    rng = random.Random(11)
    ctx = ctx_new()
    runs = []
    for d in range(1, 5):
        for _ in range(3):
            row = tuple(rng.choice((-1, 0, 1)) for _ in range(d))
            m = validate_model(TernaryModel(d, (DenseLayer((row,), (rng.randint(-d, d),)), SignActivation()), "sign_bits"))
            for xs in itertools.product((-1, 1), repeat=d):
                outs, _ = eval_model(ctx, m, encrypt_input(ctx, list(xs)), EvalOptions(plus_one=plus_one))
                runs.append((m, list(xs), outs))
    ctx.flush()
    for m, xs, outs in runs:
        assert decrypt_output(ctx, outs) == oracle_eval(m, xs)


def _random_dense(rng, d, p, mode, ternary, bn):
    rows = tuple(tuple(rng.choice((-1, 0, 1) if ternary else (-1, 1)) for _ in range(d)) for _ in range(p))
    layers = [DenseLayer(rows, tuple(rng.randint(-d // 2, d // 2) for _ in range(p)))]
    if bn:
        layers.append(BatchNorm(gamma=tuple(rng.choice([0.0] + [rng.uniform(-2, 2)] * 9) for _ in range(p)),
                                beta=tuple(rng.uniform(-3, 3) for _ in range(p)),
                                mu=tuple(rng.uniform(-4, 4) for _ in range(p)),
                                sigma2=tuple(rng.uniform(0.1, 6) for _ in range(p)), epsilon=0.001))
    if mode == "sign_bits":
        layers.append(SignActivation())
    return validate_model(TernaryModel(d, tuple(layers), mode))


# test_acceptance.py:117-187 (oracle equivalence on random dense / conv / two-layer models; reduced count)
def test_random_models_match_oracle_eval():
    rng = random.Random(1001)
    ctx = ctx_new()
    runs = []
    for case in range(40):
        mode = "score_words" if case % 5 == 0 else "sign_bits"
        m = _random_dense(rng, rng.randint(8, 40), rng.randint(1, 4), mode, case % 2 == 0, case % 3 == 0 and mode == "sign_bits")
        opts = EvalOptions(plus_one=case % 2 == 0, comparator="sort" if case % 4 == 3 else "reduce",
                           cache_shared_sums=case % 7 != 0)
        for _ in range(2):
            xs = [rng.choice((-1, 1)) for _ in range(m.input_shape)]
            outs, _ = eval_model(ctx, m, encrypt_input(ctx, xs), opts)
            runs.append((m, xs, outs))
    for case in range(10):
        shape = (rng.randint(1, 2), rng.randint(4, 5), rng.randint(4, 5))
        k = rng.randint(2, 3)
        filters = tuple(tuple(tuple(tuple(rng.choice((-1, 0, 1)) for _ in range(k)) for _ in range(k))
                              for _ in range(shape[0])) for _ in range(rng.randint(1, 2)))
        m = validate_model(TernaryModel(shape, (ConvLayer(filters, tuple(rng.randint(-2, 2) for _ in filters)),
                                                 SignActivation()), "sign_bits"))
        xs = [rng.choice((-1, 1)) for _ in range(shape[0] * shape[1] * shape[2])]
        outs, _ = eval_model(ctx, m, encrypt_input(ctx, xs), EvalOptions(plus_one=case % 2 == 0))
        runs.append((m, xs, outs))
    for case in range(6):
        d, h, p = rng.randint(6, 16), rng.randint(2, 6), rng.randint(1, 3)
        l1 = tuple(tuple(rng.choice((-1, 0, 1)) for _ in range(d)) for _ in range(h))
        l2 = tuple(tuple(rng.choice((-1, 0, 1)) for _ in range(h)) for _ in range(p))
        mode = "score_words" if case % 2 else "sign_bits"
        layers = [DenseLayer(l1, tuple(rng.randint(-3, 3) for _ in range(h))), SignActivation(),
                  DenseLayer(l2, tuple(rng.randint(-3, 3) for _ in range(p)))]
        if mode == "sign_bits":
            layers.append(SignActivation())
        m = validate_model(TernaryModel(d, tuple(layers), mode))
        xs = [rng.choice((-1, 1)) for _ in range(d)]
        outs, _ = eval_model(ctx, m, encrypt_input(ctx, xs), EvalOptions(plus_one=case % 2 == 0))
        runs.append((m, xs, outs))
    ctx.flush()
    for m, xs, outs in runs:
        assert decrypt_output(ctx, outs) == oracle_eval(m, xs)


def test_stats_identical_to_simcontext_on_a_model():
    rng = random.Random(5)
    m = _random_dense(rng, 64, 6, "sign_bits", True, False)
    xs = [rng.choice((-1, 1)) for _ in range(64)]
    sim, ctx = SimContext(), ctx_new()
    o1, s1 = eval_model(sim, m, encrypt_input(sim, xs))
    o2, s2 = eval_model(ctx, m, encrypt_input(ctx, xs))
    assert sim.global_stats.as_dict() == ctx.global_stats.as_dict()
    assert [ls.total for ls in s1.layers] == [ls.total for ls in s2.layers]
    assert decrypt_output(ctx, o2) == decrypt_output(sim, o1)


def test_shipped_cancer_model_on_gpu():
    from hebnn.wire import parse_model

    model = parse_model(json.load(open(os.path.join(HERE, "golden", "cancer_model.json"))))
    rng = random.Random(17)
    ctx = ctx_new()
    runs = []
    for _ in range(4):
        xs = [rng.choice((-1, 1)) for _ in range(model.input_shape)]
        outs, _ = eval_model(ctx, model, encrypt_input(ctx, xs))
        runs.append((xs, outs))
    for xs, outs in runs:
        assert decrypt_output(ctx, outs) == oracle_eval(model, xs)


def test_cfg2_single_neuron_784():
    """BASELINE.json configs[1]: one 784->1 neuron (+-1 weights, bias 0, sign)."""
    rng = random.Random(0)
    row = tuple(rng.choice((-1, 1)) for _ in range(784))
    model = validate_model(TernaryModel(784, (DenseLayer((row,), (0,)), SignActivation()), "sign_bits"))
    xs = [rng.choice((-1, 1)) for _ in range(784)]
    ctx = ctx_new()
    outs, _ = eval_model(ctx, model, encrypt_input(ctx, xs))
    assert decrypt_output(ctx, outs) == oracle_eval(model, xs)
    assert 9000 < ctx.gate_count < 11000


def test_lanes_batch_of_inputs_share_one_dag():
    """f1 lane batching: 8 inputs through one DAG == 8 separate oracle_evals."""
    rng = random.Random(3)
    d, p, lanes = 48, 4, 8
    rows = tuple(tuple(rng.choice((-1, 1)) for _ in range(d)) for _ in range(p))
    model = validate_model(TernaryModel(d, (DenseLayer(rows, (0,) * p),), "score_words"))
    X = np.array([[rng.choice((0, 1)) for _ in range(d)] for _ in range(lanes)], np.uint8)
    ctx = ctx_new(lanes=lanes)
    xb = ctx.encrypt_many(X.T)
    outs, _ = eval_model(ctx, model, xb)
    for w in outs:
        bits = ctx.decrypt_many(w.bits)  # [width][lanes]
        vals = (bits.astype(np.int64) << np.arange(len(w.bits))[:, None]).sum(axis=0)
        width = len(w.bits)
        vals = np.where(vals >= 1 << (width - 1), vals - (1 << width), vals) if w.signed else vals
        w._vals = vals
    for lane in range(lanes):
        xs = [1 if b else -1 for b in X[lane]]
        assert [int(w._vals[lane]) for w in outs] == oracle_eval(model, xs)


def test_replay_cached_dag_on_gpu():
    """f1 per-model DAG caching: one DAG, several encrypted inputs."""
    from hebnn.compiler import encrypt_input

    rng = random.Random(8)
    d, p = 64, 5
    rows = tuple(tuple(rng.choice((-1, 0, 1)) for _ in range(d)) for _ in range(p))
    m = validate_model(TernaryModel(d, (DenseLayer(rows, (0,) * p), SignActivation()), "sign_bits"))
    ctx = ctx_new()
    xs = [rng.choice((-1, 1)) for _ in range(d)]
    xb = encrypt_input(ctx, xs)
    outs, _ = eval_model(ctx, m, xb)
    assert decrypt_output(ctx, outs) == oracle_eval(m, xs)
    for trial in range(3):
        xs2 = [rng.choice((-1, 1)) for _ in range(d)]
        ctx.replay(xb, ctx.keys.encrypt([1 if v == 1 else 0 for v in xs2], seed=50 + trial))
        assert decrypt_output(ctx, outs) == oracle_eval(m, xs2)


@pytest.mark.parametrize("config", ["cfg2n", "cfg2l", "cfg3", "cfg4", "cfg5", "conv"])
def test_baseline_configs_full_size(config, tmp_path):
    """Every BASELINE.json BNN config at full size (cfg2n: one 784-input neuron;
    cfg2l: the 784->256 layer; cfg3: 784-256-256-10, batch 8; cfg4: its
    80%-sparse ternary variant; cfg5: tabular 240-128-64-2, batch 64; conv: an
    MNIST-shaped conv BNN through conv_layer, compiler.py:372-416) through
    the reference compiler (compiler.py:441-462) on the default context
    (streaming flushes, narrow-level deferral, full-adder and half-adder
    fusion): every output equals oracle_eval (model.py:458-497) on the first
    evaluation, when the DAG is replayed on a second encrypted batch, and when
    a fresh context runs the compiled schedule (saved and reloaded) on a third;
    counted stats are the reference SimContext's and fusion executes fewer
    bootstraps than it counts."""
    from paper_1806_03461_b200 import workloads

    # the two largest configs skip the compiled-schedule leg (a third full evaluation, ~50 s of
    # device time; the other four cover it) to keep the GPU tier inside its time limit
    cached = config not in ("cfg3", "cfg5")
    rep = workloads.run_encrypted(TfheContext, config, seed=0, replays=1, cached=cached,
                                  schedule_path=str(tmp_path / f"{config}.sched.npz"))
    assert rep["matches_oracle_eval"] is True
    assert rep["replay"]["matches_oracle_eval"] is True
    assert not cached or rep["cached"]["matches_oracle_eval"] is True
    model, batch = workloads.build(config, 0)
    sim = workloads.run_sim_reference(config, seed=0)
    assert rep["counted_gates_per_input"] == sim["counted_gates_per_input"]
    assert rep["executed_bootstraps"] < 0.45 * rep["counted_gates"]
