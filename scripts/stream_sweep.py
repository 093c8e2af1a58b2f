"""First-evaluation latency of a BNN config for several streaming settings
(stream_at, stream_min_width), each run twice in one warm process.
Usage: python scripts/stream_sweep.py [config]"""
import functools
import json
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__)))]
sys.path.insert(1, os.path.join(sys.path[0], "baseline", "_ref"))
from paper_1806_03461_b200 import workloads  # noqa: E402
from paper_1806_03461_b200.backend import TfheContext  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2l"
warm = TfheContext(seed=0)
warm.decrypt(warm.g_and(warm.encrypt(1), warm.encrypt(1)))
workloads.run_encrypted(TfheContext, cfg)  # grow pools once
for sa in (8192, 16384, 32768):
    for w in (0, 296, 592, 1184):
        ctx_cls = functools.partial(TfheContext, stream_at=sa, stream_min_width=w)
        runs = [workloads.run_encrypted(ctx_cls, cfg) for _ in range(2)]
        print(json.dumps({"stream_at": sa, "min_width": w, "first_eval_s": [round(r["first_eval_s"], 3) for r in runs],
                          "levels": [r["levels"] for r in runs], "ok": all(r["matches_oracle_eval"] for r in runs)}),
              flush=True)
