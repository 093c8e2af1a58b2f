"""Where a replay's time goes: wall time of a replay vs the sum of its levels'
kernel times (CUDA events per level, measured in a second, synchronised replay).
Usage: python scripts/replay_trace.py [cfg2n|cfg2l|...] [--graph]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "baseline", "_ref")]
import numpy as np  # noqa: E402

from hebnn.compiler import EvalOptions, eval_model  # noqa: E402
from paper_1806_03461_b200 import backend as B  # noqa: E402
from paper_1806_03461_b200 import workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2n"
warm = B.TfheContext(seed=0)
warm.decrypt(warm.g_and(warm.encrypt(1), warm.encrypt(1)))
model, batch = workloads.build(cfg, 0)
X = workloads.inputs(cfg, model, batch, 1)
ctx = B.TfheContext(seed=0, lanes=batch)
xb = ctx.encrypt_many(X.T)
outs, _ = eval_model(ctx, model, xb, EvalOptions())
got = workloads.decode_outputs(ctx, outs)
cts = ctx.keys.encrypt(X.reshape(-1), seed=5, stream=77).reshape(batch, X.shape[1], -1).transpose(1, 0, 2)
walls = []
for _ in range(3):
    t0 = time.perf_counter()
    ctx.replay(xb, cts)
    walls.append(time.perf_counter() - t0)
sched = ctx._replay_schedule()
eng = ctx._ensure_engine()
per = []
for lvl, recs in sched:
    eng.sync()
    t0 = time.perf_counter()
    eng.run_gates(recs, lanes=batch)
    br, ks = eng.last_timing()
    per.append({"level": lvl, "records": int(recs.size), "br_ms": br, "ks_ms": ks,
                "host_ms": 1e3 * (time.perf_counter() - t0)})
kern = sum(p["br_ms"] + p["ks_ms"] for p in per)
print(json.dumps({"config": cfg, "levels": len(sched), "replay_wall_ms": [1e3 * w for w in walls],
                  "sum_kernel_ms": kern, "per_level": per}))
