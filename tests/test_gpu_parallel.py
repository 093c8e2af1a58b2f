"""Out-P on real ciphertexts: two ranks (gloo process group, both on cuda:0 —
their kernels never wait on each other) each evaluate half of every layer's
output units on the B200 and all-gather the layer's output ciphertexts;
decrypted scores equal oracle_eval."""

import os
import random
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "baseline", "_ref")]
    import numpy as np
    import torch.distributed as dist

    from hebnn.model import DenseLayer, SignActivation, TernaryModel, oracle_eval, validate_model
    from paper_1806_03461_b200.backend import TfheContext, shared_keys
    from paper_1806_03461_b200.parallel import OutPEvaluator, TorchComm, decode_scores

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = random.Random(12)
        d, h, p = 64, 9, 4
        l1 = tuple(tuple(rng.choice((-1, 1)) for _ in range(d)) for _ in range(h))
        l2 = tuple(tuple(rng.choice((-1, 0, 1)) for _ in range(h)) for _ in range(p))
        model = validate_model(TernaryModel(d, (DenseLayer(l1, (0,) * h), SignActivation(),
                                                DenseLayer(l2, (1,) * p)), "score_words"))
        xs = [rng.choice((-1, 1)) for _ in range(d)]
        keys = shared_keys(42)
        cts = keys.encrypt(np.array([1 if v == 1 else 0 for v in xs], np.uint8), seed=8, stream=3)
        ev = OutPEvaluator(lambda: TfheContext(seed=42), TorchComm(device="cpu"))
        words = ev.run(model, cts[:, None, :])
        scores = [int(v) for v in decode_scores(TfheContext(seed=42), words)[0]]
        q.put((rank, scores == oracle_eval(model, xs), scores, [s["units"] for s in ev.stats]))
    finally:
        dist.destroy_process_group()


def test_outp_two_ranks_on_gpu():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        rank, ok, scores, units = q.get(timeout=600)
        res[rank] = (ok, scores, units)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res[0][0] and res[1][0]
    assert res[0][1] == res[1][1]
    assert res[0][2][0][0] == 0 and res[0][2][0][1] == res[1][2][0][0] and res[1][2][0][1] == 9


def test_bench_two_ranks_sharing_the_gpu():
    """`bench.py --gpus 2` spawns its two ranks itself; with HB_BENCH_SHARE_GPU=1
    both run on cuda:0 over gloo: the line says n_gpus 2, the NAND outputs are
    right, the strong-scaling leg splits the job, and Out-P on the cfg2 neuron
    and batch sharding of cfg5 match oracle_eval."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, HB_BENCH_SHARE_GPU="1")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3", "--gates", "512",
                        "--bnn", "cfg2n,cfg5", "--no-compare", "--no-cpu-baseline"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["correct"] is True
    assert d["strong_scaling"]["gates_per_gpu"] == 256 and d["strong_scaling"]["n_gpus"] == 2
    assert d["bnn"]["cfg2n"]["matches_oracle_eval"] is True, d["bnn"]["cfg2n"]
    assert d["bnn"]["cfg5"]["matches_oracle_eval"] is True, d["bnn"]["cfg5"]
    # the same two legs with the carry-save popcount on both ranks
    assert d["bnn_csa"]["cfg2n"]["matches_oracle_eval"] is True, d["bnn_csa"]["cfg2n"]
    assert d["bnn_csa"]["cfg5"]["matches_oracle_eval"] is True, d["bnn_csa"]["cfg5"]
    assert d["bnn_csa"]["cfg5"]["executed_bootstraps_this_rank"] < 0.7 * d["bnn"]["cfg5"]["executed_bootstraps_this_rank"]
