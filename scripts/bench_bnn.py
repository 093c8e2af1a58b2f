"""Encrypted-BNN latency for BASELINE.json configs 2-5 on one B200 (through
the reference compiler on TfheContext).  Usage: python scripts/bench_bnn.py cfg2n cfg2l cfg3 ..."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "baseline", "_ref")]
from paper_1806_03461_b200 import workloads  # noqa: E402
from paper_1806_03461_b200.backend import TfheContext  # noqa: E402

warm = TfheContext(seed=0)
warm.decrypt(warm.g_and(warm.encrypt(1), warm.encrypt(1)))  # CUDA context, keys, engine
for cfg in sys.argv[1:] or ["cfg2n"]:
    rep = workloads.run_encrypted(TfheContext, cfg, replays=1)
    print(json.dumps(rep), flush=True)
