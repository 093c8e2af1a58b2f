"""Streaming flushes on the B200: background level batches while the
reference compiler builds the DAG give bit-identical output ciphertexts (same
plaintexts when a flush boundary splits a half-adder pair)."""

import random

import numpy as np
import pytest

from hebnn.compiler import eval_model
from hebnn.model import DenseLayer, SignActivation, TernaryModel, oracle_eval, validate_model

pytestmark = pytest.mark.gpu


def test_streaming_flush_bit_identical():
    from paper_1806_03461_b200.backend import TfheContext

    rng = random.Random(3)
    d, p = 200, 12
    rows = tuple(tuple(rng.choice((-1, 1)) for _ in range(d)) for _ in range(p))
    model = validate_model(TernaryModel(d, (DenseLayer(rows, (0,) * p), SignActivation()), "sign_bits"))
    xs = [rng.choice((0, 1)) for _ in range(d)]
    want = oracle_eval(model, [1 if v else -1 for v in xs])
    # A gate's output ciphertext is a function of its input ciphertexts only, whatever batch
    # it runs in — except for the half-adder pairing, which fuses an XOR and an AND only when
    # both are in the same flush: a background flush that starts between the two gate calls of
    # a half adder (timing-dependent) runs them unfused, with the same plaintexts but other
    # ciphertext bits.  Bit identity is therefore checked without the pairing, plaintext
    # identity with it.
    for fuse in (False, True):
        outs = []
        for stream_at, width in ((0, 0), (300, 0), (300, 64)):
            ctx = TfheContext(seed=42, enc_stream=77, stream_at=stream_at, stream_min_width=width,
                              fuse_half_adders=fuse)
            handles = [ctx.encrypt(v) for v in xs]
            res, _ = eval_model(ctx, model, handles)
            outs.append((ctx.export_ciphertexts(res), [ctx.decrypt(h) for h in res], ctx.exec_stats["flushes"]))
        for o in outs[1:]:  # streamed (all levels / wide levels only) == one flush
            if not fuse:
                assert np.array_equal(outs[0][0], o[0])  # bit for bit
            assert outs[0][1] == o[1]
        assert [1 if b else -1 for b in outs[0][1]] == want
        assert outs[1][2] > outs[0][2]
