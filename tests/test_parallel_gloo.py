"""Out-P multi-rank evaluation (parallel.py) with world_size 2 over gloo on
CPU: each rank evaluates its share of every layer's output units on its own
(plaintext stand-in) engine and the layer outputs are all-gathered as
ciphertexts; results must equal the reference oracle_eval and a single-rank
run."""

import os
import random
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q, csa=False):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "baseline", "_ref"), os.path.join(root, "tests")]
    import torch.distributed as dist

    from hebnn.model import DenseLayer, SignActivation, TernaryModel, oracle_eval, validate_model
    from paper_1806_03461_b200.parallel import OutPEvaluator, TorchComm, decode_scores
    from plain_engine import plain_context_class

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Ctx = plain_context_class()
        rng = random.Random(5)
        d, h, p = 24, 7, 3
        l1 = tuple(tuple(rng.choice((-1, 0, 1)) for _ in range(d)) for _ in range(h))
        l2 = tuple(tuple(rng.choice((-1, 1)) for _ in range(h)) for _ in range(p))
        results = {}
        for mode in ("sign_bits", "score_words"):
            layers = [DenseLayer(l1, tuple(rng.randint(-2, 2) for _ in range(h))), SignActivation(),
                      DenseLayer(l2, tuple(rng.randint(-2, 2) for _ in range(p)))]
            if mode == "sign_bits":
                layers.append(SignActivation())
            model = validate_model(TernaryModel(d, tuple(layers), mode))
            xs = [rng.choice((-1, 1)) for _ in range(d)]
            enc = Ctx(seed=42)
            cts = enc.keys.encrypt(np.array([1 if v == 1 else 0 for v in xs], np.uint8), seed=3, stream=9)
            ev = OutPEvaluator(lambda: Ctx(seed=42, csa_popcount=csa), TorchComm())
            out = ev.run(model, cts[:, None, :])
            if mode == "sign_bits":
                bits = enc.keys.decrypt(np.stack(out)[:, 0, :])
                got = [1 if b else -1 for b in bits]
            else:
                got = [int(v) for v in decode_scores(enc, out)[0]]
            results[mode] = (got == oracle_eval(model, xs), got, [s["units"] for s in ev.stats])
        q.put((rank, results))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,csa", [(2, False), (2, True)])
def test_outp_two_ranks_gloo(world, csa):
    """csa: every rank's contexts use the opt-in carry-save popcount (popcount.py)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, csa)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(world):
        for mode, (ok, got, units) in res[rank].items():
            assert ok, (rank, mode, got)
            assert units[0][0] <= units[0][1]
    assert {m: v[1] for m, v in res[0].items()} == {m: v[1] for m, v in res[1].items()}


def test_partition_balances_cost():
    from paper_1806_03461_b200.parallel import partition

    assert partition(7, 2) == [(0, 4), (4, 7)]
    # one expensive unit first: cost-balanced split puts it alone
    parts = partition(5, 2, costs=[10, 1, 1, 1, 1])
    assert parts == [(0, 1), (1, 5)]
    parts = partition(10, 4, costs=[1] * 10)
    assert sum(h - l for l, h in parts) == 10 and all(h >= l for l, h in parts)
    assert partition(2, 4, costs=[1, 1])[-1][1] == 2
