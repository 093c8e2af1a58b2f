"""Host-side behaviour of TfheContext (the GateBackend drop-in) without a GPU:
the SimContext contract (backend.py:161-257) for stats, levels, scopes,
errors and handle identity, and the DAG lowering (elision, CSE, hb_gate
record encoding) executed on a plaintext stand-in engine and compared with
the reference SimContext on the same circuits."""

import random
import threading

import pytest

from hebnn import backend as ref_backend
from hebnn.backend import AND, COSTED_KINDS, MUX, OR, XNOR, XOR, CipherBit, ContextMismatchError, ScopeError, SimContext
from hebnn.circuits import compare_ge_const, decrypt_word, encrypt_word, rc_add, rc_sub, reduce_tree_sum
from hebnn.compiler import EvalOptions, decrypt_output, encrypt_input, eval_model
from hebnn.model import DenseLayer, SignActivation, TernaryModel, oracle_eval, validate_model
from paper_1806_03461_b200.backend import TfheContext
from plain_engine import plain_context_class

Plain = plain_context_class()
PLAIN_FN = {AND: lambda a, b: a & b, OR: lambda a, b: a | b, XOR: lambda a, b: a ^ b, XNOR: lambda a, b: 1 - (a ^ b)}


def gate(ctx, kind):
    return {AND: ctx.g_and, OR: ctx.g_or, XOR: ctx.g_xor, XNOR: ctx.g_xnor}[kind]


def test_is_a_reference_gate_backend():
    ctx = Plain(seed=42)
    assert isinstance(ctx, ref_backend.GateBackend)
    assert isinstance(ctx.encrypt(1), CipherBit)


def test_encrypt_and_trivial_reject_non_bits():
    ctx = Plain(seed=42)
    with pytest.raises(ValueError):
        ctx.encrypt(2)
    with pytest.raises(ValueError):
        ctx.trivial_const(-1)


def test_counts_levels_histogram_like_simcontext():
    ctx = Plain(seed=42)
    a, b = ctx.encrypt(1), ctx.encrypt(0)
    out = ctx.g_and(a, b)
    assert ctx.global_stats.counts[AND] == 1 and out.level == 1
    deeper = ctx.g_or(out, b)
    assert deeper.level == 2
    assert ctx.global_stats.level_histogram == {1: 1, 2: 1}


def test_trivial_and_not_are_free():
    ctx = Plain(seed=42)
    for _ in range(50):
        ctx.trivial_const(1)
    a = ctx.encrypt(1)
    for _ in range(7):
        a = ctx.g_not(a)
    assert ctx.gate_count == 0
    assert ctx.g_not(a).level == a.level
    assert ctx.g_not(ctx.trivial_const(0)).trivial_value == 1
    assert ctx.g_not(ctx.encrypt(0)).trivial_value is None
    assert ctx.decrypt(a) == 0


def test_not_priced_as_xnor_when_switch_off(monkeypatch):
    monkeypatch.setattr(ref_backend, "NOT_IS_FREE", False)
    ctx = Plain(seed=42)
    a = ctx.encrypt(1)
    na = ctx.g_not(a)
    assert ctx.global_stats.counts[XNOR] == 1 and na.level == 1
    assert ctx.decrypt(na) == 0


def test_foreign_handles_rejected():
    c1, c2 = Plain(seed=42), Plain(seed=42)
    bit = c1.encrypt(1)
    with pytest.raises(ContextMismatchError):
        c2.decrypt(bit)
    with pytest.raises(ContextMismatchError):
        c2.g_and(bit, c2.encrypt(1))
    with pytest.raises(ContextMismatchError):
        c1.g_and(bit, "not a bit")
    sim = SimContext()
    with pytest.raises(ContextMismatchError):
        c1.g_xor(bit, sim.encrypt(1))


def test_mux_trivial_selector_returns_same_handle():
    ctx = Plain(seed=42)
    x, y = ctx.encrypt(1), ctx.encrypt(0)
    assert ctx.g_mux(ctx.trivial_const(1), x, y) is x
    assert ctx.g_mux(ctx.trivial_const(0), x, y) is y
    assert ctx.gate_count == 0


def test_scopes():
    ctx = Plain(seed=42)
    ctx.begin_scope("empty")
    st = ctx.end_scope()
    assert st.total == 0 and st.max_level == 0 and st.label == "empty"
    a, b = ctx.encrypt(1), ctx.encrypt(1)
    ctx.begin_scope("ha")
    ctx.g_xor(a, b)
    ctx.g_and(a, b)
    assert ctx.scope_depth == 1
    st = ctx.end_scope()
    assert st.counts == {AND: 1, OR: 0, XOR: 1, XNOR: 0, MUX: 0} and st.max_level == 1
    with pytest.raises(ScopeError):
        ctx.end_scope()


def _random_circuit(ctx, rng, inputs, n):
    bits = list(inputs)
    for _ in range(n):
        op = rng.choice(["and", "or", "xor", "xnor", "not", "mux", "const"])
        a, b = rng.choice(bits), rng.choice(bits)
        if op == "not":
            bits.append(ctx.g_not(a))
        elif op == "mux":
            bits.append(ctx.g_mux(rng.choice(bits), a, b))
        elif op == "const":
            bits.append(ctx.trivial_const(rng.randint(0, 1)))
        else:
            bits.append(getattr(ctx, f"g_{op}")(a, b))
    return bits


@pytest.mark.parametrize("seed", range(12))
def test_random_dags_match_simcontext_values_and_stats(seed):
    """Same random circuit (incl. trivial constants, repeated inputs, MUX,
    NOT) on SimContext and TfheContext: decrypted values, levels and stats
    agree; elision/CSE executes fewer gates than counted."""
    values = [random.Random(seed).randint(0, 1) for _ in range(5)]
    sim, ctx = SimContext(), Plain(seed=42)
    sb = _random_circuit(sim, random.Random(100 + seed), [sim.encrypt(v) for v in values], 60)
    cb = _random_circuit(ctx, random.Random(100 + seed), [ctx.encrypt(v) for v in values], 60)
    assert [b.level for b in sb] == [b.level for b in cb]
    assert [b.trivial_value for b in sb] == [b.trivial_value for b in cb]
    assert [sim.decrypt(b) for b in sb] == [ctx.decrypt(b) for b in cb]
    assert sim.global_stats.as_dict() == ctx.global_stats.as_dict()
    assert ctx.exec_stats["gates"] <= ctx.gate_count


def test_circuits_and_models_match_oracle_on_plain_engine():
    ctx = Plain(seed=42)
    for x in range(16):
        for y in range(16):
            assert decrypt_word(rc_add(encrypt_word(ctx, x, 4), encrypt_word(ctx, y, 4))) == x + y
    assert decrypt_word(rc_sub(encrypt_word(ctx, 3, 3), encrypt_word(ctx, 5, 3))) == -2
    word = reduce_tree_sum([ctx.encrypt(b) for b in (1, 0, 1, 1, 1, 0, 1)])
    assert decrypt_word(word) == 5
    assert ctx.decrypt(compare_ge_const(word, 5)) == 1 and ctx.decrypt(compare_ge_const(word, 6)) == 0
    rng = random.Random(9)
    for trial in range(4):
        d, p = rng.randint(8, 40), rng.randint(1, 4)
        rows = tuple(tuple(rng.choice((-1, 0, 1)) for _ in range(d)) for _ in range(p))
        mode = "score_words" if trial % 2 else "sign_bits"
        layers = (DenseLayer(rows, tuple(rng.randint(-3, 3) for _ in range(p))),)
        if mode == "sign_bits":
            layers += (SignActivation(),)
        m = validate_model(TernaryModel(d, layers, mode))
        xs = [rng.choice((-1, 1)) for _ in range(d)]
        for opts in (EvalOptions(), EvalOptions(plus_one=False), EvalOptions(comparator="sort")):
            c = Plain(seed=42)
            outs, _ = eval_model(c, m, encrypt_input(c, xs), opts)
            assert decrypt_output(c, outs) == oracle_eval(m, xs)


def test_lanes_share_one_dag():
    ctx = Plain(seed=42, lanes=4)
    a = ctx.encrypt_lanes([0, 1, 0, 1])
    b = ctx.encrypt_lanes([0, 0, 1, 1])
    assert list(ctx.decrypt(ctx.g_and(a, b))) == [0, 0, 0, 1]
    assert list(ctx.decrypt(ctx.g_xor(a, b))) == [0, 1, 1, 0]
    assert list(ctx.decrypt(ctx.g_mux(a, b, ctx.g_not(b)))) == [1, 0, 0, 1]
    assert ctx.gate_count == 3


def test_concurrent_gate_issue_is_race_free():
    ctx = Plain(seed=42)
    inputs = [ctx.encrypt(i % 2) for i in range(8)]

    def work(seed):
        rng = random.Random(seed)
        for _ in range(200):
            ctx.g_and(rng.choice(inputs), rng.choice(inputs))

    threads = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert ctx.global_stats.counts[AND] == 800
    assert sum(ctx.global_stats.level_histogram.values()) == 800


def test_flush_requires_a_device_on_the_product_context():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1806_03461_b200.backend import DeviceError

    ctx = TfheContext(seed=42)
    x = ctx.g_and(ctx.encrypt(1), ctx.encrypt(1))
    with pytest.raises(DeviceError):
        ctx.decrypt(x)


def test_all_costed_kinds_present():
    assert COSTED_KINDS == (AND, OR, XOR, XNOR, MUX)


def test_replay_reuses_the_dag_for_new_inputs():
    """f1: evaluate once, then replay the recorded schedule on new inputs."""
    rng = random.Random(21)
    d, p = 20, 3
    rows = tuple(tuple(rng.choice((-1, 1)) for _ in range(d)) for _ in range(p))
    m = validate_model(TernaryModel(d, (DenseLayer(rows, (0,) * p), SignActivation()), "sign_bits"))
    ctx = Plain(seed=42)
    xs = [rng.choice((-1, 1)) for _ in range(d)]
    xb = encrypt_input(ctx, xs)
    outs, _ = eval_model(ctx, m, xb)
    assert decrypt_output(ctx, outs) == oracle_eval(m, xs)
    gates_before = ctx.gate_count
    for trial in range(3):
        xs2 = [rng.choice((-1, 1)) for _ in range(d)]
        cts = ctx.keys.encrypt([1 if v == 1 else 0 for v in xs2], seed=100 + trial)
        ctx.replay(xb, cts)
        assert decrypt_output(ctx, outs) == oracle_eval(m, xs2)
    assert ctx.gate_count == gates_before  # no new DAG nodes
