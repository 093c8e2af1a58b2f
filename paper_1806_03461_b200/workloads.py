"""Seeded synthetic workloads of BASELINE.json configs 2-5 (encrypted BNNs).

MNIST and the tabular datasets are not in the container; inputs are synthetic
with the shapes and distributions BASELINE.json states (Bernoulli(0.5) bits;
uniform 8-bit feature values), weights uniform +-1 (or ternary with a
Bernoulli(0.8) zero mask for cfg4), biases 0, all from `random.Random(seed)`.
"""

from __future__ import annotations

import os
import random
import time

import numpy as np

from hebnn.compiler import EvalOptions, eval_model
from hebnn.model import ConvLayer, DenseLayer, SignActivation, TernaryModel, oracle_eval, validate_model


def _dense(rng, d, p, zero_prob=0.0):
    rows = []
    for _ in range(p):
        row = []
        for _ in range(d):
            w = rng.choice((-1, 1))
            if zero_prob and rng.random() < zero_prob:
                w = 0
            row.append(w)
        rows.append(tuple(row))
    return DenseLayer(tuple(rows), (0,) * p)


def _conv(rng, out_c, in_c, k, stride=1, zero_prob=0.0):
    filters = []
    for _ in range(out_c):
        filt = []
        for _ in range(in_c):
            filt.append(tuple(tuple(0 if (zero_prob and rng.random() < zero_prob) else rng.choice((-1, 1))
                                    for _ in range(k)) for _ in range(k)))
        filters.append(tuple(filt))
    return ConvLayer(tuple(filters), (0,) * out_c, stride=stride)


def build(config, seed=0):
    """Returns (model, batch) for config in {cfg2n, cfg2l, cfg3, cfg4, cfg5, conv}.

    conv (not a BASELINE config): an MNIST-shaped convolutional
    BNN through the reference's conv_layer (compiler.py:372-416) — 1x28x28 bits,
    conv 5x5 8 ch stride 1 + sign (24x24), conv 5x5 16 ch stride 2 + sign
    (10x10), dense 1600 -> 10 score words; +-1 weights; one input."""
    rng = random.Random(seed)
    if config == "conv":
        layers = (_conv(rng, 8, 1, 5), SignActivation(), _conv(rng, 16, 8, 5, stride=2), SignActivation(),
                  _dense(rng, 1600, 10))
        return validate_model(TernaryModel((1, 28, 28), layers, "score_words")), 1
    if config == "cfg2n":
        return validate_model(TernaryModel(784, (_dense(rng, 784, 1), SignActivation()), "sign_bits")), 1
    if config == "cfg2l":
        return validate_model(TernaryModel(784, (_dense(rng, 784, 256), SignActivation()), "sign_bits")), 1
    if config in ("cfg3", "cfg4"):
        z = 0.8 if config == "cfg4" else 0.0
        layers = (_dense(rng, 784, 256, z), SignActivation(), _dense(rng, 256, 256, z), SignActivation(),
                  _dense(rng, 256, 10, z))
        return validate_model(TernaryModel(784, layers, "score_words")), 8
    if config == "cfg5":
        layers = (_dense(rng, 240, 128), SignActivation(), _dense(rng, 128, 64), SignActivation(), _dense(rng, 64, 2))
        return validate_model(TernaryModel(240, layers, "score_words")), 64
    raise ValueError(f"unknown config {config!r}")


def inputs(config, model, batch, seed=1):
    """[batch][d] bits in {0,1} (stored-binary encoding of +-1 inputs)."""
    rng = np.random.default_rng(seed)
    d = int(np.prod(model.input_shape))
    if config == "cfg5":
        vals = rng.integers(0, 256, (batch, 30))  # 30 features quantised to 8 bits
        return ((vals[:, :, None] >> np.arange(8)[None, None, :]) & 1).reshape(batch, d).astype(np.uint8)
    return rng.integers(0, 2, (batch, d)).astype(np.uint8)


def flatten_outputs(outs):
    """eval_model outputs -> (flat handle list, structure): sign bits, or score
    words as [(width, signed)] (compiler.py EncryptedWord)."""
    if outs and hasattr(outs[0], "bits"):
        return [b for w in outs for b in w.bits], [(len(w.bits), bool(w.signed)) for w in outs]
    return list(outs), None


def decode_bits(bits, structure):
    """Decrypted flat output bits [handles][lanes] -> [lanes][units]: sign bits
    -> +-1, score words -> ints (two's complement when signed)."""
    if structure is None:
        return np.where(np.asarray(bits).T == 1, 1, -1)
    cols, at = [], 0
    for width, signed in structure:
        wb = np.asarray(bits[at:at + width]).astype(np.int64)
        at += width
        v = (wb << np.arange(width)[:, None]).sum(axis=0)
        if signed:
            v = np.where(v >= 1 << (width - 1), v - (1 << width), v)
        cols.append(v)
    return np.stack(cols, axis=1)


def decode_outputs(ctx, outs):
    """Decrypt eval_model outputs for every lane: sign bits -> +-1, words -> ints.
    Returns [lanes][units]."""
    flat, structure = flatten_outputs(outs)
    return decode_bits(ctx.decrypt_many(flat), structure)


def run_cached(ctx_cls, config, sched, structure, seed=0, device=0, check=True, trial=0):
    """First evaluation of a fresh context from a compiled schedule (no reference
    compiler, no gate DAG): encrypt a new batch, run every level, decrypt."""
    model, batch = build(config, seed)
    X = inputs(config, model, batch, seed + 200 + trial)
    ctx = ctx_cls(seed=seed, device=device, lanes=batch)
    t0 = time.perf_counter()
    cts = ctx.keys.encrypt(X.reshape(-1), seed=seed + 11, stream=600 + trial).reshape(batch, X.shape[1], -1)
    cts = np.ascontiguousarray(cts.transpose(1, 0, 2))
    t1 = time.perf_counter()
    out = ctx.run_schedule(sched, cts)
    t2 = time.perf_counter()
    bits = ctx.keys.decrypt(out.reshape(-1, out.shape[-1])).reshape(out.shape[0], batch)
    got = decode_bits(bits, structure)
    t3 = time.perf_counter()
    ok = None
    if check:
        ok = all(list(got[b]) == oracle_eval(model, [1 if v else -1 for v in X[b]]) for b in range(batch))
    return {"first_eval_s": t3 - t0, "encrypt_s": t1 - t0, "run_s": t2 - t1, "decrypt_s": t3 - t2,
            "levels": len(sched.levels), "records": sched.records, "matches_oracle_eval": ok}


GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def cancer_rows(path=None):
    """The reference's shipped Cancer dataset, binned exactly as its trainer
    does (tests/golden/make_cancer_fixture.py): (bits [569][90] stored-binary,
    labels +-1, train idx, test idx, (train acc, test acc) from metrics.json)."""
    z = np.load(path or os.path.join(GOLDEN, "cancer_rows.npz"))
    return (z["bits"], z["labels"], z["train"], z["test"],
            (float(z["accuracy_train"]), float(z["accuracy_test"])))


def cancer_model(path=None):
    """The reference's shipped trained model (trainer/out/model.json)."""
    from hebnn.wire import read_model

    return read_model(path or os.path.join(GOLDEN, "cancer_model.json"))


def run_cancer(ctx_cls, seed=0, device=0, rows=None, check=True):
    """Classify the Cancer rows encrypted, all of them as lanes of one DAG
    (the shipped 90-input model through the reference compiler); predictions
    checked row by row against oracle_eval, accuracy against metrics.json."""
    X, y, train, test, (acc_train, acc_test) = cancer_rows()
    if rows is not None:
        X, y = X[rows], y[rows]
    model = cancer_model()
    ctx = ctx_cls(seed=seed, device=device, lanes=X.shape[0])
    t0 = time.perf_counter()
    xb = ctx.encrypt_many(X.T)
    outs, _ = eval_model(ctx, model, xb, EvalOptions())
    got = decode_outputs(ctx, outs)[:, 0]
    dt = time.perf_counter() - t0
    rep = {"rows": int(X.shape[0]), "latency_s": dt, "rows_per_s": X.shape[0] / dt,
           "counted_gates_per_row": ctx.gate_count, "executed_bootstraps": ctx.exec_stats["bootstraps"],
           "predictions": got}
    if check:
        want = np.array([oracle_eval(model, [1 if v else -1 for v in row])[0] for row in X])
        rep["matches_oracle_eval"] = bool(np.array_equal(got, want))
    if rows is None:
        rep["accuracy_train"] = float((got[train] == y[train]).mean())
        rep["accuracy_test"] = float((got[test] == y[test]).mean())
        rep["trainer_accuracy"] = {"train": acc_train, "test": acc_test}
    return rep


def run_sim_reference(config, seed=0, options=EvalOptions()):
    """The reference's own CPU path for the same workload: SimContext +
    eval_model (plaintext gate simulation, backend.py:162-237 and
    compiler.py eval_model), one input.  Reported beside the encrypted run."""
    from hebnn.backend import SimContext

    model, batch = build(config, seed)
    X = inputs(config, model, batch, seed + 1)
    ctx = SimContext()
    t0 = time.perf_counter()
    xs = [ctx.encrypt(int(v)) for v in X[0]]
    outs, _ = eval_model(ctx, model, xs, options)
    dt = time.perf_counter() - t0
    return {"kind": "reference SimContext (plaintext, 1 thread)", "inputs": 1, "seconds_per_input": dt,
            "counted_gates_per_input": ctx.gate_count, "counted_gates_per_s": ctx.gate_count / dt}


def run_encrypted(ctx_cls, config, seed=0, device=0, options=EvalOptions(), check=True, replays=0, cached=False,
                  schedule_path=None):
    """Encrypt a batch, evaluate through the reference compiler on a
    lane-batched context, decrypt, compare with oracle_eval.  Returns a report.
    cached: also compile the executed schedule (saved to / reloaded from
    `schedule_path` when given) and time a fresh context's first evaluation
    through it (report key "cached")."""
    model, batch = build(config, seed)
    X = inputs(config, model, batch, seed + 1)
    ctx = ctx_cls(seed=seed, device=device, lanes=batch)
    t0 = time.perf_counter()
    xb = ctx.encrypt_many(X.T)
    t1 = time.perf_counter()
    outs, _ = eval_model(ctx, model, xb, options)
    t2 = time.perf_counter()
    ctx.flush()
    t3 = time.perf_counter()
    got = decode_outputs(ctx, outs)
    t4 = time.perf_counter()
    ok = None
    if check:
        ok = all(list(got[b]) == oracle_eval(model, [1 if v else -1 for v in X[b]]) for b in range(batch))
    counted = ctx.gate_count * batch
    replay = None
    if replays:
        # steady-state serving: new encrypted batch through the cached DAG
        times, oks = [], []
        for r in range(replays):
            X2 = inputs(config, model, batch, seed + 100 + r)
            cts = ctx.keys.encrypt(X2.reshape(-1), seed=seed + 7, stream=500 + r).reshape(
                batch, X2.shape[1], -1).transpose(1, 0, 2)
            ta = time.perf_counter()
            ctx.replay(xb, cts)
            got2 = decode_outputs(ctx, outs)
            times.append(time.perf_counter() - ta)
            if check:
                oks.append(all(list(got2[b]) == oracle_eval(model, [1 if v else -1 for v in X2[b]])
                               for b in range(batch)))
        replay = {"replays": replays, "latency_s": min(times), "bootstraps_per_s": ctx.exec_stats["bootstraps"] / min(times),
                  "matches_oracle_eval": all(oks) if check else None}
    cached_rep = None
    if cached:
        from .backend import Schedule

        flat, structure = flatten_outputs(outs)
        tc = time.perf_counter()
        sched = ctx.compile_schedule(xb, flat, meta={"config": config})
        compile_s = time.perf_counter() - tc
        if schedule_path:
            sched.save(schedule_path)
            sched = Schedule.load(schedule_path)
        cached_rep = run_cached(ctx_cls, config, sched, structure, seed=seed, device=device, check=check)
        cached_rep["compile_s"] = compile_s
    return {
        "config": config, "batch": batch, "counted_gates": counted,
        "counted_gates_per_input": ctx.gate_count,
        "executed_bootstraps": ctx.exec_stats["bootstraps"], "levels": ctx.exec_stats["levels"],
        "depth": ctx.global_stats.max_level,
        # first evaluation: encrypt + DAG build through the reference compiler (with
        # background flushes running on the device meanwhile) + final flush + decrypt
        "first_eval_s": t4 - t0,
        "encrypt_s": t1 - t0, "dag_build_s": t2 - t1, "final_flush_s": t3 - t2, "decrypt_s": t4 - t3,
        "background_flushes": ctx.exec_stats["flushes"] - 1,
        "bootstraps_per_s": ctx.exec_stats["bootstraps"] / (t4 - t0),
        "counted_gates_per_s": counted / (t4 - t0),
        "matches_oracle_eval": ok,
        "replay": replay,
        "cached": cached_rep,
    }
