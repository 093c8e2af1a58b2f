"""Decrypted-bit semantics of the exact CPU oracle pinned against the
reference: the reference's own checks (truth tables, MUX, half adder, adders,
an exhaustive small neuron — test_backend.py:52-58,116-123,
test_circuits.py:36-82, test_compiler.py:150-165) replayed on TfheContext
with every flush executed by the oracle on real CGGI ciphertexts (CPU, no GPU).
Circuits are built first and decrypted together, so each level is one batch."""

import itertools

import pytest

from hebnn.backend import AND, MUX, OR, XNOR, XOR
from hebnn.circuits import decrypt_word, encrypt_word, half_adder, rc_add
from hebnn.compiler import EvalOptions, decrypt_output, encrypt_input, eval_model
from hebnn.model import DenseLayer, SignActivation, TernaryModel, oracle_eval, validate_model
from oracle_engine import oracle_context_class

Ctx = oracle_context_class()
PLAIN = {AND: lambda a, b: a & b, OR: lambda a, b: a | b, XOR: lambda a, b: a ^ b, XNOR: lambda a, b: 1 - (a ^ b)}


def test_gate_truth_tables_exhaustive():
    ctx = Ctx(seed=42)
    cases = []
    for kind in (AND, OR, XOR, XNOR):
        fn = {AND: ctx.g_and, OR: ctx.g_or, XOR: ctx.g_xor, XNOR: ctx.g_xnor}[kind]
        for a, b in itertools.product((0, 1), repeat=2):
            cases.append((kind, a, b, fn(ctx.encrypt(a), ctx.encrypt(b))))
    got = ctx.decrypt_many([h for *_, h in cases])[:, 0]
    assert [int(v) for v in got] == [PLAIN[k](a, b) for k, a, b, _ in cases]
    assert ctx.exec_stats["bootstraps"] == 16


def test_mux_exhaustive_native_two_bootstraps():
    ctx = Ctx(seed=42)
    outs, want = [], []
    for s, a, b in itertools.product((0, 1), repeat=3):
        outs.append(ctx.g_mux(ctx.encrypt(s), ctx.encrypt(a), ctx.encrypt(b)))
        want.append(a if s else b)
    assert [int(v) for v in ctx.decrypt_many(outs)[:, 0]] == want
    assert ctx.global_stats.counts[MUX] == 8
    assert ctx.exec_stats["bootstraps"] == 16  # native CGGI MUX: 2 blind rotations each


def test_half_adder_and_two_bit_adder():
    ctx = Ctx(seed=42)
    has = [(a, b, half_adder(ctx.encrypt(a), ctx.encrypt(b))) for a, b in itertools.product((0, 1), repeat=2)]
    sums = [(x, y, rc_add(encrypt_word(ctx, x, 2), encrypt_word(ctx, y, 2))) for x, y in ((1, 2), (3, 3))]
    for a, b, (s, c) in has:
        assert (ctx.decrypt(s), ctx.decrypt(c)) == ((a + b) % 2, (a + b) // 2)
    for x, y, w in sums:
        assert decrypt_word(w) == x + y


@pytest.mark.parametrize("plus_one", [True, False])
def test_small_neuron_exhaustive_matches_oracle_eval(plus_one):
    model = validate_model(TernaryModel(3, (DenseLayer(((1, -1, 1),), (0,)), SignActivation()), "sign_bits"))
    ctx = Ctx(seed=42)
    runs = []
    for xs in itertools.product((-1, 1), repeat=3):
        outs, _ = eval_model(ctx, model, encrypt_input(ctx, list(xs)), EvalOptions(plus_one=plus_one))
        runs.append((list(xs), outs))
    for xs, outs in runs:
        assert decrypt_output(ctx, outs) == oracle_eval(model, xs)
