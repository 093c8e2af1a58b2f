"""First-evaluation latency with and without streaming flushes (one B200).
Usage: python scripts/stream_ab.py cfg2l cfg3 [threshold ...]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "baseline", "_ref")]
from paper_1806_03461_b200 import workloads  # noqa: E402
from paper_1806_03461_b200.backend import TfheContext  # noqa: E402

warm = TfheContext(seed=0)
warm.decrypt(warm.g_and(warm.encrypt(1), warm.encrypt(1)))
cfgs = [a for a in sys.argv[1:] if not a.isdigit()] or ["cfg2l"]
thresholds = [int(a) for a in sys.argv[1:] if a.isdigit()] or [0, 16384]
for cfg in cfgs:
    for sa in thresholds:
        cls = type("C", (TfheContext,), {"__init__": lambda self, *a, _sa=sa, **k: TfheContext.__init__(self, *a, stream_at=_sa, **k)})
        rep = workloads.run_encrypted(cls, cfg)
        print(json.dumps({"config": cfg, "stream_at": sa, "first_eval_s": rep["first_eval_s"],
                          "dag_build_s": rep["dag_build_s"], "final_flush_s": rep["final_flush_s"],
                          "executed": rep["executed_bootstraps"], "levels": rep["levels"],
                          "ok": rep["matches_oracle_eval"]}), flush=True)
