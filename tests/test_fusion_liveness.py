"""Host DAG: full-adder fusion into 3-input bootstraps (majority, XOR3) and
the live-handle filter of flush (dormant gates), on the plaintext stand-in
engine (CPU).  Decrypted values and GateStats must equal SimContext's."""

import itertools

import numpy as np

from hebnn.backend import SimContext
from hebnn.circuits import encrypt_word, decrypt_word, rc_add, reduce_tree_sum
from plain_engine import plain_context_class

Ctx = plain_context_class()


def _fa(ctx, a, b, c):
    # reference circuits._full_adder (circuits.py:101-108)
    axb = ctx.g_xor(a, b)
    s = ctx.g_xor(axb, c)
    t = ctx.g_and(axb, c)
    return s, ctx.g_or(ctx.g_and(a, b), t)


def test_full_adder_is_two_bootstraps_and_exact():
    for bits in itertools.product((0, 1), repeat=3):
        ctx = Ctx(seed=3)
        a, b, c = (ctx.encrypt(v) for v in bits)
        s, cout = _fa(ctx, a, b, c)
        assert (ctx.decrypt(s), ctx.decrypt(cout)) == (sum(bits) & 1, int(sum(bits) >= 2))
        assert ctx.exec_stats["bootstraps"] == 2  # XOR3 + MAJ; the 3 intermediates stay dormant
        assert ctx.gate_count == 5                # counted like SimContext
        assert ctx.exec_stats["levels"] == 1


def test_full_adder_with_negated_inputs():
    for bits in itertools.product((0, 1), repeat=3):
        ctx = Ctx(seed=3)
        a, b, c = (ctx.encrypt(v) for v in bits)
        na, nc = ctx.g_not(a), ctx.g_not(c)
        s, cout = _fa(ctx, na, b, nc)
        x = (1 - bits[0], bits[1], 1 - bits[2])
        assert (ctx.decrypt(s), ctx.decrypt(cout)) == (sum(x) & 1, int(sum(x) >= 2))


def test_live_intermediate_is_still_executed():
    ctx = Ctx(seed=4)
    a, b, c = ctx.encrypt(1), ctx.encrypt(0), ctx.encrypt(1)
    axb = ctx.g_xor(a, b)
    s = ctx.g_xor(axb, c)
    t = ctx.g_and(axb, c)
    cout = ctx.g_or(ctx.g_and(a, b), t)
    assert ctx.decrypt(cout) == 1 and ctx.decrypt(s) == 0
    assert ctx.decrypt(t) == 1 and ctx.decrypt(axb) == 1  # were live: executed in the same flush


def test_dormant_gate_is_revived_by_cse_and_by_reuse():
    ctx = Ctx(seed=5)
    a, b = ctx.encrypt(1), ctx.encrypt(1)
    ctx.g_and(a, b)                  # handle dropped at once
    keep = ctx.g_xor(a, b)
    assert ctx.decrypt(keep) == 0
    before = ctx.exec_stats["bootstraps"]
    again = ctx.g_and(a, b)          # CSE hit on the dormant AND
    assert ctx.decrypt(again) == 1
    assert ctx.exec_stats["bootstraps"] == before + 1
    # a dormant operand deep in a new gate
    x = ctx.g_and(a, ctx.g_not(b))   # dormant after the next flush
    y = ctx.g_or(x, a)
    del x
    assert ctx.decrypt(y) == 1


def test_stats_and_values_match_simcontext_on_adder_trees():
    rng = np.random.default_rng(7)
    for trial in range(4):
        n = int(rng.integers(3, 12))
        vals = rng.integers(0, 2, n).tolist()
        outs = []
        for C in (SimContext, lambda: Ctx(seed=9)):
            ctx = C()
            bits = [ctx.encrypt(v) for v in vals]
            w = reduce_tree_sum(bits)
            x = rc_add(w, encrypt_word(ctx, 5, w.width))
            outs.append((decrypt_word(w), decrypt_word(x), ctx.global_stats.as_dict()))
        assert outs[0] == outs[1]
        assert outs[0][0] == sum(vals)


def test_native_live_filter_matches_python_walk():
    """The native DAG's live-gate filter (hb_dag.cpp) equals a plain graph walk
    from the nodes holding live handles through pending operands."""
    ctx = Ctx(seed=11, stream_at=0)
    rng = np.random.default_rng(3)
    bits = [ctx.encrypt(int(v)) for v in rng.integers(0, 2, 300)]
    w = reduce_tree_sum(bits)
    keep = [w.bits[-1], ctx.g_and(bits[0], bits[1])]
    del w
    dag = ctx._dag
    pend = dag.pending()
    op, a, b, c, _ = dag.gather(pend)
    fields = {int(n): (int(o), int(x) >> 1, int(y) >> 1, int(z) >> 1) for n, o, x, y, z in zip(pend, op, a, b, c)}
    stack = [n for n in fields if dag.hcount(n) > 0]
    need = set()
    while stack:
        n = stack.pop()
        if n in need:
            continue
        need.add(n)
        for m in fields[n][1:]:
            if m in fields and m not in need:
                stack.append(m)
    assert sorted(dag.live(False).tolist()) == sorted(need)
    assert 0 < len(need) < len(fields)
    assert keep


def test_streaming_flush_matches_single_flush():
    """Background flushes while the DAG is built (stream_at) give the same
    values and stats; only a few extra gates (live at the trigger) may run."""
    rng = np.random.default_rng(12)
    vals = rng.integers(0, 2, 300).tolist()
    res = []
    for stream_at in (0, 200):
        ctx = Ctx(seed=13, stream_at=stream_at, stream_min_width=0)
        bits = [ctx.encrypt(v) for v in vals]
        w = reduce_tree_sum(bits)
        x = rc_add(w, encrypt_word(ctx, 77, w.width))
        res.append((decrypt_word(w), decrypt_word(x), ctx.global_stats.as_dict(), ctx.exec_stats["bootstraps"],
                    ctx.exec_stats["flushes"]))
    assert res[0][:3] == res[1][:3] and res[0][0] == sum(vals)
    assert res[1][4] > 1                        # background flushes happened
    assert res[1][3] <= res[0][3] * 1.05        # little extra work


def test_concurrent_gate_issue_with_streaming():
    """Several threads issue gates on one context (SimContext's lock contract,
    backend.py:174,200) while background flushes run (small stream_at)."""
    import threading

    ctx = Ctx(seed=21, stream_at=64, stream_min_width=0)
    rng = np.random.default_rng(5)
    data = [rng.integers(0, 2, 40).tolist() for _ in range(4)]
    results = {}

    def work(i):
        bits = [ctx.encrypt(v) for v in data[i]]
        results[i] = reduce_tree_sum(bits)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    for i in range(4):
        assert decrypt_word(results[i]) == sum(data[i])
    assert ctx.exec_stats["flushes"] > 1


def test_streaming_defers_narrow_levels():
    """stream_min_width: a background flush runs only levels with enough
    bootstraps whose operands are done or run with them; the rest stay
    pending (values and stats unchanged, fewer and wider launches)."""
    rng = np.random.default_rng(31)
    vals = [rng.integers(0, 2, 120).tolist() for _ in range(6)]
    res = []
    for width in (0, 24):
        ctx = Ctx(seed=17, stream_at=150, stream_min_width=width)
        words = []
        for v in vals:
            words.append(reduce_tree_sum([ctx.encrypt(x) for x in v]))
        got = [decrypt_word(w) for w in words]
        res.append((got, ctx.global_stats.as_dict(), ctx.exec_stats["levels"], ctx.exec_stats["flushes"]))
    assert res[0][:2] == res[1][:2] and res[0][0] == [sum(v) for v in vals]
    assert res[1][3] > 1                 # background flushes still happened
    assert res[1][2] < res[0][2]         # and the narrow levels were merged


def test_select_wide_respects_dependencies():
    """Every gate _select_wide runs has its operands done or run with it, every
    run level is wide enough, and run + deferred is the live pending set."""
    ctx = Ctx(seed=19, stream_at=0, stream_min_width=20)
    rng = np.random.default_rng(4)
    words = [reduce_tree_sum([ctx.encrypt(int(x)) for x in rng.integers(0, 2, n)]) for n in (90, 40, 7)]
    dag = ctx._dag
    live = dag.live(False)
    run, deferred = ctx._select_wide(live)
    assert sorted(np.concatenate([run, deferred]).tolist()) == sorted(live.tolist())
    assert run.size > 0 and deferred.size > 0
    runset = set(run.tolist())
    op, a, b, c, lvl = dag.gather(run)
    for x in (a, b, c):
        for m in (x >> 1).tolist():
            assert m == 0 or dag.is_done(m) or m in runset
    _, counts = np.unique(lvl, return_counts=True)
    assert counts.min() >= 20
    assert words
