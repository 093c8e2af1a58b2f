"""Half-adder fusion on the host (CPU): the oracle's one-rotation half adder
(oracle/tfhe_oracle.c or_half_adder) against the truth table and the plain AND
gate, and TfheContext's pairing of XOR / AND-of-literals nodes into HA records
(decrypted results and GateStats unchanged, one bootstrap per half adder)."""

import os

import numpy as np
import pytest

from oracle import oracle as O

ORACLE_SO = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_build",
                         "libtfhe_oracle.so")
pytestmark = pytest.mark.skipif(not os.path.exists(ORACLE_SO), reason="oracle not built (make -C oracle)")

EIGHTH = 1 << 29


def test_oracle_half_adder_truth_table_and_and_output():
    p = O.default_params()
    k = O.Keys(p, 5)
    c = O.Context(p, k)
    for a in (0, 1):
        for b in (0, 1):
            ca = O.encrypt(p, k, np.array([a], np.uint8), 1, 1)[0]
            cb = O.encrypt(p, k, np.array([b], np.uint8), 1, 2)[0]
            for al in (1, -1):
                for be in (1, -1):
                    la, lb = (a if al > 0 else 1 - a), (b if be > 0 else 1 - b)
                    for sg in (1, -1):
                        oa, ox = c.half_adder((-EIGHTH) & 0xFFFFFFFF, al, ca, be, cb, sg)
                        da, dx = O.decrypt(p, k, np.stack([oa, ox]))
                        assert da == (la & lb)
                        assert dx == ((la ^ lb) if sg > 0 else 1 - (la ^ lb))
                        # the AND output is the plain AND gate, bit for bit (same rotation and extraction)
                        assert np.array_equal(oa, c.gate((-EIGHTH) & 0xFFFFFFFF, al, ca, be, cb))


def _ctx(cls_factory, **kw):
    return cls_factory()(seed=3, stream_at=0, **kw)


def test_context_fuses_half_adders_oracle_engine():
    """reference circuits.half_adder on real ciphertexts (CPU oracle engine):
    one bootstrap per half adder, same decrypted bits and stats as unfused."""
    from hebnn.circuits import half_adder
    from oracle_engine import oracle_context_class

    res = []
    for fuse in (True, False):
        ctx = _ctx(oracle_context_class, fuse_half_adders=fuse)
        out = []
        for a in (0, 1):
            for b in (0, 1):
                s, cy = half_adder(ctx.encrypt(a), ctx.encrypt(b))
                # OR and XNOR of the same pair pair up too (AND of negated literals / negated XOR)
                o = ctx.g_or(ctx.encrypt(a), ctx.encrypt(b))
                out.append((s, cy, o))
        ctx.flush()
        vals = [(ctx.decrypt(s), ctx.decrypt(cy)) for s, cy, _ in out]
        res.append((vals, ctx.global_stats.as_dict(), ctx.exec_stats["bootstraps"],
                    ctx.exec_stats.get("half_adders", 0)))
    assert res[0][0] == res[1][0] == [(0, 0), (1, 0), (1, 0), (0, 1)]
    assert res[0][1] == res[1][1]
    assert res[0][3] == 4 and res[1][3] == 0
    assert res[0][2] == res[1][2] - 4


def test_context_half_adder_signs_plain_engine():
    """Every literal-sign combination of an AND/OR paired with XOR/XNOR of the
    same two nodes (plaintext stand-in engine, exhaustive inputs)."""
    from plain_engine import plain_context_class

    ctx = _ctx(plain_context_class)
    cases = []
    for a in (0, 1):
        for b in (0, 1):
            x, y = ctx.encrypt(a), ctx.encrypt(b)
            for na in (False, True):
                for nb in (False, True):
                    la = ctx.g_not(x) if na else x
                    lb = ctx.g_not(y) if nb else y
                    want_a, want_b = (1 - a if na else a), (1 - b if nb else b)
                    cases.append((ctx.g_and(la, lb), want_a & want_b))
                    cases.append((ctx.g_or(la, lb), want_a | want_b))
            cases.append((ctx.g_xor(x, y), a ^ b))
            cases.append((ctx.g_xnor(x, y), 1 - (a ^ b)))
    sched = ctx.schedule()
    kinds = np.concatenate([r["kind"] for _, r in sched])
    assert np.count_nonzero(kinds == 3) == 4  # one HA per input pair
    ctx.flush()
    assert [ctx.decrypt(h) for h, _ in cases] == [w for _, w in cases]
