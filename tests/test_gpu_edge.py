"""Edge cases of the engine and the drop-in on the GPU: invalid records,
empty levels, pool growth preserving contents, native MUX across lanes,
NOT priced as XNOR, concurrent contexts sharing one engine."""

import threading

import numpy as np
import pytest

from hebnn import backend as ref_backend
from paper_1806_03461_b200 import tfhe
from paper_1806_03461_b200.backend import TfheContext

pytestmark = pytest.mark.gpu


def test_invalid_records_are_value_errors(engine, keys):
    engine.reserve(8)
    recs = tfhe.gate_records(1)
    recs[0] = (2, 0, 1, 0, 0, 1, 1, 7, 0)  # unknown kind
    with pytest.raises(ValueError, match="kind"):
        engine.run_gates(recs)
    recs[0] = (10 ** 9, 0, 1, 0, 0, 1, 1, 0, 0)  # slot beyond capacity
    with pytest.raises(ValueError, match="capacity"):
        engine.run_gates(recs)
    recs[0] = (2, 0, 1, 5, 0, 1, 1, 3, 0)  # half adder without an XOR orientation (gamma 0)
    with pytest.raises(ValueError, match="HA record"):
        engine.run_gates(recs)
    recs[0] = (2, 0, 1, 2, 0, 1, 1, 3, 1)  # half adder writing both outputs to one slot
    with pytest.raises(ValueError, match="HA record"):
        engine.run_gates(recs)
    engine.run_gates(tfhe.gate_records(0))  # empty level is a no-op
    engine.sync()


def test_pool_growth_while_levels_are_queued(keys):
    """Stream-ordered pool growth between queued levels and async copies:
    slots written before the growth keep their values, levels after it see
    them, async uploads issued before it land in the new allocation."""
    eng = tfhe.Engine(keys)
    n = 600
    rng = np.random.default_rng(11)
    a, b = rng.integers(0, 2, n).astype(np.uint8), rng.integers(0, 2, n).astype(np.uint8)
    eng.reserve(5 * n)
    eng.upload(0, np.concatenate([keys.encrypt(a, seed=1, stream=1), keys.encrypt(b, seed=1, stream=2)]))
    recs = tfhe.gate_records(n)
    c0, al, be = tfhe.GATE_LIN["AND"]
    recs["dst"], recs["src_a"], recs["src_b"] = np.arange(2 * n, 3 * n), np.arange(n), np.arange(n, 2 * n)
    recs["c0"], recs["alpha"], recs["beta"] = c0, al, be
    eng.run_gates(recs)                        # queued on the engine stream
    c = rng.integers(0, 2, n).astype(np.uint8)
    eng.upload_async(3 * n, keys.encrypt(c, seed=1, stream=3))
    eng.reserve(50_000)                        # grows while the level (and the copy) may still run
    recs2 = tfhe.gate_records(n)
    c0, al, be = tfhe.GATE_LIN["XOR"]
    recs2["dst"], recs2["src_a"], recs2["src_b"] = np.arange(4 * n, 5 * n), np.arange(2 * n, 3 * n), np.arange(n)
    recs2["c0"], recs2["alpha"], recs2["beta"] = c0, al, be
    eng.run_gates(recs2)
    eng.sync()
    assert np.array_equal(keys.decrypt(eng.download(2 * n, n)), a & b)
    assert np.array_equal(keys.decrypt(eng.download(4 * n, n)), (a & b) ^ a)
    assert np.array_equal(keys.decrypt(eng.download(3 * n, n)), c)
    eng.close()


def test_pool_growth_preserves_contents(keys):
    eng = tfhe.Engine(keys)
    cts = keys.encrypt(np.array([1, 0, 1], np.uint8), seed=3)
    eng.reserve(3)
    eng.upload(0, cts)
    eng.reserve(200_000)  # grow: old slots copied into the new allocation
    assert eng.capacity >= 200_000
    assert np.array_equal(eng.download(0, 3), cts)
    eng.close()


def test_native_mux_across_lanes():
    lanes = 8
    ctx = TfheContext(seed=42, lanes=lanes)
    rng = np.random.default_rng(1)
    S, A, B = (rng.integers(0, 2, lanes) for _ in range(3))
    s, a, b = (ctx.encrypt_lanes(v) for v in (S, A, B))
    m = ctx.g_mux(s, a, ctx.g_not(b))
    assert list(ctx.decrypt(m)) == list(np.where(S == 1, A, 1 - B))
    assert ctx.exec_stats["bootstraps"] == 2 * lanes  # one native MUX = 2 blind rotations per lane


def test_not_priced_as_xnor_on_gpu(monkeypatch):
    monkeypatch.setattr(ref_backend, "NOT_IS_FREE", False)
    ctx = TfheContext(seed=42)
    a = ctx.encrypt(1)
    na = ctx.g_not(a)
    assert ctx.global_stats.counts["XNOR"] == 1
    assert ctx.decrypt(na) == 0 and ctx.decrypt(ctx.g_not(na)) == 1


def test_concurrent_contexts_share_one_engine():
    errors = []

    def work(seed):
        try:
            ctx = TfheContext(seed=42)
            rng = np.random.default_rng(seed)
            bits = rng.integers(0, 2, (16, 2))
            outs = [ctx.g_xor(ctx.encrypt(int(x)), ctx.encrypt(int(y))) for x, y in bits]
            got = ctx.decrypt_many(outs)[:, 0]
            if list(got) != list(bits[:, 0] ^ bits[:, 1]):
                errors.append(seed)
        except Exception as exc:  # pragma: no cover - reported below
            errors.append(repr(exc))

    threads = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert errors == []


def test_async_double_buffered_transfers(keys):
    """hb_pool_upload_async / hb_pool_download_async overlapping consecutive
    levels on two slot regions give the same results as synchronous copies."""
    import torch

    eng = tfhe.Engine(keys)
    n, words = 64, keys.params.n + 1
    rng = np.random.default_rng(9)
    steps = 5
    bits = [rng.integers(0, 2, 2 * n).astype(np.uint8) for _ in range(steps)]
    h_in = [torch.empty((2 * n, words), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32) for _ in range(steps)]
    h_out = [torch.empty((n, words), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32) for _ in range(steps)]
    for k in range(steps):
        h_in[k][:] = keys.encrypt(bits[k], seed=20 + k)
    eng.reserve(6 * n)
    c0, al, be = tfhe.GATE_LIN["XOR"]
    recs = []
    for r in range(2):
        rc = tfhe.gate_records(n)
        rc["dst"], rc["src_a"], rc["src_b"] = 3 * n * r + 2 * n + np.arange(n), 3 * n * r + np.arange(n), 3 * n * r + n + np.arange(n)
        rc["c0"], rc["alpha"], rc["beta"] = c0, al, be
        recs.append(rc)
    for k in range(steps):
        r = k % 2
        eng.upload_async(3 * n * r, h_in[k])
        eng.run_gates(recs[r])
        eng.download_async(3 * n * r + 2 * n, h_out[k])
    eng.sync()
    for k in range(steps):
        assert np.array_equal(keys.decrypt(h_out[k]), bits[k][:n] ^ bits[k][n:]), k
    eng.close()


@pytest.mark.gpu
def test_async_download_is_not_overtaken_by_later_levels(keys):
    """Write-after-read: step k's async download (a long copy, its gate outputs at
    the end of the range) must read step k's values even though step k+2 rewrites
    the same slots with a short level right after (hb_engine.cu WAR)."""
    import torch

    eng = tfhe.Engine(keys)
    g, span, words = 8, 32768, keys.params.n + 1
    steps = 4
    rng = np.random.default_rng(21)
    bits = [rng.integers(0, 2, 2 * g).astype(np.uint8) for _ in range(steps)]
    h_in = [keys.encrypt(bits[k], seed=40 + k) for k in range(steps)]
    h_out = [torch.empty((span, words), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32) for _ in range(steps)]
    region = span + 2 * g
    eng.reserve(2 * region)
    c0, al, be = tfhe.GATE_LIN["AND"]
    recs = []
    for r in range(2):
        base = r * region
        rc = tfhe.gate_records(g)
        # outputs in the LAST g slots of the downloaded span, inputs after it
        rc["dst"] = base + span - g + np.arange(g)
        rc["src_a"], rc["src_b"] = base + span + np.arange(g), base + span + g + np.arange(g)
        rc["c0"], rc["alpha"], rc["beta"] = c0, al, be
        recs.append(rc)
    for k in range(steps):
        r = k % 2
        eng.upload(r * region + span, h_in[k])
        eng.run_gates(recs[r])
        eng.download_async(r * region, h_out[k])
    eng.sync()
    for k in range(steps):
        got = keys.decrypt(h_out[k][span - g:])
        assert np.array_equal(got, bits[k][:g] & bits[k][g:]), k
    eng.close()


@pytest.mark.gpu
def test_async_download_fences_are_range_aware_and_survive_many_downloads(keys):
    """More async downloads than the engine tracks individually (8): the older
    ones are folded into one fenced range, and a later level rewriting the slots
    of the FIRST download must still wait for it; levels writing other slots do
    not (their results are checked too)."""
    import torch

    eng = tfhe.Engine(keys)
    g, span, words = 8, 8192, keys.params.n + 1
    steps = 12
    rng = np.random.default_rng(33)
    bits = [rng.integers(0, 2, 2 * g).astype(np.uint8) for _ in range(steps + 1)]
    region = span + 2 * g
    eng.reserve((steps + 1) * region)
    h_out = [torch.empty((span, words), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
             for _ in range(steps)]
    c0, al, be = tfhe.GATE_LIN["AND"]

    h_in = [torch.empty((2 * g, words), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
            for _ in range(steps + 1)]
    for k in range(steps + 1):
        h_in[k][:] = keys.encrypt(bits[k], seed=60 + k)

    def level(r, k):
        base = r * region
        eng.upload_async(base + span, h_in[k])  # range-aware fences only (no full fence)
        rc = tfhe.gate_records(g)
        rc["dst"] = base + span - g + np.arange(g)
        rc["src_a"], rc["src_b"] = base + span + np.arange(g), base + span + g + np.arange(g)
        rc["c0"], rc["alpha"], rc["beta"] = c0, al, be
        eng.run_gates(rc)

    for k in range(steps):
        level(k, k)
        eng.download_async(k * region, h_out[k])
    level(0, steps)  # rewrites the outputs of the first (folded) download
    eng.sync()
    for k in range(steps):
        got = keys.decrypt(h_out[k][span - g:])
        assert np.array_equal(got, bits[k][:g] & bits[k][g:]), k
    now = keys.decrypt(eng.download(span - g, g))
    assert np.array_equal(now, bits[steps][:g] & bits[steps][g:])
    eng.close()
