import sys, time, json
sys.path[:0] = ['/root/repo', '/root/repo/baseline/_ref']
import numpy as np
from paper_1806_03461_b200 import workloads
from paper_1806_03461_b200 import backend as B
from hebnn.compiler import eval_model, EvalOptions

log = []
orig_launch = B.TfheContext._launch
orig_run = B.TfheContext._run_batches
T0 = [0]
def launch(self, wait):
    t = time.perf_counter()
    orig_launch(self, wait)
    log.append(("launch", wait, round(t - T0[0], 3), round(time.perf_counter() - T0[0], 3), self.exec_stats["bootstraps"]))
def run(eng, batches, lanes, errors):
    t = time.perf_counter()
    orig_run(eng, batches, lanes, errors)
    log.append(("bg_done", len(batches), round(t - T0[0], 3), round(time.perf_counter() - T0[0], 3), sum(len(r) for _, r in batches)))
B.TfheContext._launch = launch
B.TfheContext._run_batches = staticmethod(run)
warm = B.TfheContext(seed=0); warm.decrypt(warm.g_and(warm.encrypt(1), warm.encrypt(1)))
CFG = sys.argv[1] if len(sys.argv) > 1 else 'cfg2l'
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    log.clear()
    model, batch = workloads.build(CFG, 0)
    X = workloads.inputs(CFG, model, batch, 1)
    ctx = B.TfheContext(seed=0, lanes=batch)
    T0[0] = time.perf_counter()
    xb = ctx.encrypt_many(X.T)
    outs, _ = eval_model(ctx, model, xb, EvalOptions())
    t_build = time.perf_counter() - T0[0]
    ctx.flush()
    t_all = time.perf_counter() - T0[0]
    print('rep', rep, 'build', round(t_build, 3), 'total', round(t_all, 3))
    for e in log: print('  ', e)
