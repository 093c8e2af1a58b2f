"""Compiled level schedules ("compile once, serve many"):
TfheContext.compile_schedule / run_schedule / Schedule.save+load, on the
plaintext stand-in engine (host logic only).  The GPU twin runs the BASELINE
configs through it (tests/test_gpu_configs.py)."""

import random

import numpy as np
import pytest

from hebnn.compiler import EvalOptions, eval_model
from hebnn.model import DenseLayer, SignActivation, TernaryModel, oracle_eval, validate_model
from paper_1806_03461_b200 import workloads
from paper_1806_03461_b200.backend import Schedule
from plain_engine import plain_context_class

Plain = plain_context_class()


def _model(rng, d, h, p, mode):
    l1 = tuple(tuple(rng.choice((-1, 0, 1)) for _ in range(d)) for _ in range(h))
    l2 = tuple(tuple(rng.choice((-1, 0, 1)) for _ in range(h)) for _ in range(p))
    layers = [DenseLayer(l1, tuple(rng.randint(-3, 3) for _ in range(h))), SignActivation(),
              DenseLayer(l2, tuple(rng.randint(-3, 3) for _ in range(p)))]
    if mode == "sign_bits":
        layers.append(SignActivation())
    return validate_model(TernaryModel(d, tuple(layers), mode))


def _encrypt_batch(ctx, X, seed):
    batch, d = X.shape
    cts = ctx.keys.encrypt(X.reshape(-1), seed=seed).reshape(batch, d, -1)
    return np.ascontiguousarray(cts.transpose(1, 0, 2))


@pytest.mark.parametrize("mode", ["sign_bits", "score_words"])
@pytest.mark.parametrize("lanes", [1, 3])
def test_compiled_schedule_runs_on_a_fresh_context(tmp_path, mode, lanes):
    rng = random.Random(7 if mode == "sign_bits" else 8)
    m = _model(rng, 14, 5, 3, mode)
    nrng = np.random.default_rng(3)
    X = nrng.integers(0, 2, (lanes, 14)).astype(np.uint8)
    ctx = Plain(seed=42, lanes=lanes)
    xb = ctx.encrypt_many(X.T)
    outs, _ = eval_model(ctx, m, xb, EvalOptions())
    flat, structure = workloads.flatten_outputs(outs)
    sched = ctx.compile_schedule(xb, flat, meta={"case": mode})
    assert sched.meta["counted"] == ctx.global_stats.as_dict()
    path = tmp_path / "model.sched.npz"
    sched.save(path)
    back = Schedule.load(path)
    assert back.records == sched.records and len(back.levels) == len(sched.levels)
    fresh = Plain(seed=42, lanes=lanes)
    for trial in range(3):
        X2 = nrng.integers(0, 2, (lanes, 14)).astype(np.uint8)
        out = fresh.run_schedule(back, _encrypt_batch(fresh, X2, 50 + trial))
        bits = fresh.keys.decrypt(out.reshape(-1, out.shape[-1])).reshape(out.shape[0], lanes)
        got = workloads.decode_bits(bits, structure)
        for b in range(lanes):
            assert list(got[b]) == oracle_eval(m, [1 if v else -1 for v in X2[b]]), (trial, b)
    assert fresh.gate_count == 0  # no DAG was built


def test_schedule_outputs_with_not_flags_and_constants():
    ctx = Plain(seed=42)
    a, b = ctx.encrypt(1), ctx.encrypt(0)
    x = ctx.g_and(a, b)
    outs = [x, ctx.g_not(x), ctx.trivial_const(1), ctx.trivial_const(0), ctx.g_not(a), a]
    assert [ctx.decrypt(o) for o in outs] == [0, 1, 1, 0, 0, 1]
    sched = ctx.compile_schedule([a, b], outs)
    fresh = Plain(seed=42)
    for va, vb in ((0, 0), (0, 1), (1, 0), (1, 1)):
        cts = fresh.keys.encrypt([va, vb], seed=va * 2 + vb)
        got = fresh.keys.decrypt(fresh.run_schedule(sched, cts).reshape(len(outs), -1))
        assert list(got) == [va & vb, 1 - (va & vb), 1, 0, 1 - va, va]


def test_schedule_rejects_bad_inputs(tmp_path):
    ctx = Plain(seed=42)
    a, b = ctx.encrypt(1), ctx.encrypt(0)
    x = ctx.g_xor(a, b)
    with pytest.raises(ValueError):
        ctx.compile_schedule([x], [x])  # not an input handle
    with pytest.raises(ValueError):
        ctx.compile_schedule([ctx.g_not(a)], [x])
    sched = ctx.compile_schedule([a, b], [x])
    with pytest.raises(ValueError):
        Plain(seed=42, lanes=2).run_schedule(sched, np.zeros((2, 2, 631), np.uint32))
    with pytest.raises(ValueError):
        Plain(seed=42).run_schedule(sched, np.zeros((3, 631), np.uint32))
    p = tmp_path / "bad.npz"
    sched.save(p)
    with np.load(p) as z:
        arrays = dict(z)
    arrays["sizes"] = arrays["sizes"] + 1
    np.savez(tmp_path / "bad2.npz", **arrays)
    with pytest.raises(ValueError):
        Schedule.load(tmp_path / "bad2.npz")


def test_run_encrypted_cached_leg_on_plain_engine(tmp_path):
    """workloads.run_encrypted(cached=True) (the bench's cached first evaluation),
    on the BASELINE cfg2n neuron with the stand-in engine."""
    rep = workloads.run_encrypted(Plain, "cfg2n", seed=3, cached=True, schedule_path=str(tmp_path / "s.npz"))
    assert rep["matches_oracle_eval"] and rep["cached"]["matches_oracle_eval"]
    assert rep["cached"]["records"] > 0
