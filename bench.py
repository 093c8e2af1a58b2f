#!/usr/bin/env python
"""Benchmark: bootstrapped gates/sec on B200 (BASELINE.json metric) +
encrypted-BNN latency.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[0], the metric's own micro-bench): per GPU,
4,096 independent bootstrapped NAND gates on encrypted Bernoulli(0.5) bit
pairs, keys and messages from one seed.  One step = one hb_run_gates level of
the 4,096 gates (fused gate prologue + blind rotation + sample extract, then
batched key switch) with the inputs resident in HBM.  Multi-GPU: every rank
runs its own 4,096 gates (weak scaling, replicated keys, no collective on the
data path — gates are independent), timed on the device with CUDA events and
reduced with MAX over ranks.

`e2e` repeats the step through the C ABI with host buffers: H2D of the two
input ciphertext batches from pinned memory, the gate records, the level, and
D2H of the 4,096 output ciphertexts, all inside the timed region.

`bnn` (N = 1): every BASELINE BNN config through the reference compiler on the
pure drop-in `TfheContext` (first evaluation, replay, compiled schedule, all
checked against `oracle_eval`); `bnn_csa`: the same configs with the opt-in
carry-save popcount (`TfheContext(csa_popcount=True)`, same outputs and
counted gates, ~42% fewer executed bootstraps).

`--impl reference` times the CPU path on a bounded sample of the same
workload with all host threads: the vectorised FP64-FFT CPU port of the same
gate bootstrap (oracle/tfhe_cpu_fft.c, eight gates per SIMD register, checked
bit-for-bit against the exact-integer oracle); the exact Goldilocks-NTT oracle's
own rate is reported beside it.  The reference package itself has no
ciphertext arithmetic (it simulates in plaintext).
"""

from __future__ import annotations

import argparse
import datetime
import json
import re
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
for _p in (ROOT, os.path.join(ROOT, "baseline", "_ref")):
    if _p not in sys.path:
        sys.path.insert(0, _p)

import numpy as np  # noqa: E402

# F_BS: algorithmic FP64 flops of one blind rotation.
# CGGI key (bk_unroll 1): n * [(k+1)(l+1) * F_FFT + (k+1)^2 * l * (N/2) * 8],
#   F_FFT = 5 (N/2) log2(N/2) + 6 (N/2) (transform + twist), 8 flops per complex MAC.
# Key pairs (bk_unroll 2): n/2 * [(k+1)(l+1) * F_FFT + (l * (N/2)) * (4 * (6 + 2 * 8) + 4 * 8) + 3 * (N/2) * 7]:
#   per key pair one external product; per row pair and bin the combined key
#   C_{h,o} = sum_c F_c BK_{h,c,o} (4 of them: one complex product + two complex MACs
#   each) and four complex MACs x_h C_{h,o}; F_c = (X^e_c - 1) evaluated once per
#   component and bin (complex product + subtraction).
F_FFT = 5 * 512 * 9 + 6 * 512
F_BS1 = 630 * (2 * 4 * F_FFT + 4 * 3 * 512 * 8)
F_BS2 = 315 * (2 * 4 * F_FFT + 3 * 512 * (4 * (6 + 2 * 8) + 4 * 8) + 3 * 512 * 7)
assert F_BS1 == 162_570_240 and F_BS2 == 127_249_920
F_BS = {1: F_BS1, 2: F_BS2}
METRIC = "bootstrapped gates/sec"
WORKLOAD = "cfg1: 4096 independent bootstrapped NAND gates per GPU (TFHE n=630,N=1024,k=1,Bg=2^7,l=3,KS 2^2x8)"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--gates", type=int, default=4096)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-compare", action="store_true", help="skip the CGGI-key-layout comparison leg")
    ap.add_argument("--no-csa", action="store_true", help="skip the carry-save-popcount BNN legs (bnn_csa)")
    ap.add_argument("--plan", action="store_true",
                    help="print the rank layout (n_gpus, backend, devices) as one JSON line and exit (launcher test)")
    ap.add_argument("--bnn", default="all",
                    help="encrypted-BNN latency legs (BASELINE configs 2-5), comma-separated from "
                         "cfg2n,cfg2l,cfg3,cfg4,cfg5,conv (aliases neuron, layer), 'all' or 'none': one GPU on "
                         "rank 0, or Out-P / batch sharding over all ranks for N > 1")
    args = ap.parse_args()
    alias = {"neuron": "cfg2n", "layer": "cfg2l"}
    if args.bnn == "none":
        args.bnn_list = []
    elif args.bnn == "all":
        args.bnn_list = list(BNN_CONFIGS)
    else:
        args.bnn_list = [alias.get(c, c) for c in args.bnn.split(",") if c]
        bad = [c for c in args.bnn_list if c not in BNN_CONFIGS]
        if bad:
            ap.error(f"--bnn: unknown config(s) {bad}; choose from {BNN_CONFIGS}")
    return args


BNN_CONFIGS = ("cfg2n", "cfg2l", "cfg3", "cfg4", "cfg5", "conv")


def spawn_ranks(args):
    """`python bench.py --gpus N` (N > 1) without a launcher: start the N ranks
    ourselves through torch.distributed.run (127.0.0.1 rendezvous), so the
    number of GPUs timed is always the number asked for.  Returns the exit code."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    print(f"bench.py: spawning {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


# ---------------------------------------------------------------------------
# distributed plumbing (torch.distributed: barrier + max over ranks only)
# ---------------------------------------------------------------------------

class _Rank0:
    rank = 0
    world = 1


class Dist:
    """HB_BENCH_SHARE_GPU=1 (testing only): every rank uses cuda:0 and a gloo
    process group — the ranks never wait on each other's kernels."""

    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.share = os.environ.get("HB_BENCH_SHARE_GPU") == "1"
        self.local_rank = 0 if self.share else int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.backend = None
        self.nccl_log = None
        if self.world > 1:
            import torch
            import torch.distributed as dist

            backend = "nccl" if torch.cuda.is_available() and not self.share else "gloo"
            if backend == "nccl":
                torch.cuda.set_device(self.local_rank)
                # keep NCCL's communicator lines (ring/NVLS setup) as evidence, in a file so that
                # stdout stays one JSON line; rank 0 quotes them in its line ("nccl")
                self.nccl_log = os.path.join(tempfile.gettempdir(), f"hb_bench_nccl.{os.getpid()}.log")
                os.environ.setdefault("NCCL_DEBUG", "INFO")
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
                os.environ.setdefault("NCCL_DEBUG_FILE", self.nccl_log)
            dist.init_process_group(backend=backend)
            self.backend = backend
            self.pg = dist
            self.torch = torch

    def barrier(self):
        if self.pg:
            if self.torch.cuda.is_available() and not self.share:
                self.pg.barrier(device_ids=[self.local_rank])
            else:
                self.pg.barrier()

    def max(self, x):
        if not self.pg:
            return x
        dev = f"cuda:{self.local_rank}" if self.torch.cuda.is_available() and not self.share else "cpu"
        t = self.torch.tensor([float(x)], dtype=self.torch.float64, device=dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def gather_obj(self, obj):
        if not self.pg:
            return [obj]
        out = [None] * self.world
        self.pg.all_gather_object(out, obj)
        return out

    def nccl_lines(self, limit=24):
        """This rank's NCCL INFO lines about its communicators (rings, NVLS, nRanks)."""
        path = self.nccl_log
        if not path or not os.path.exists(path):
            return []
        keep = []
        with open(path, errors="replace") as f:
            for ln in f:
                if any(k in ln for k in ("comm 0x", "NVLS", "nRanks", "Channel 00", "Connected all", "NCCL version")):
                    keep.append(ln.strip()[:200])
        return keep[:limit]

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ---------------------------------------------------------------------------
# nvidia-smi clock sampler (recipe's clocks line)
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def mark(self):
        """Start of the timed region: only samples stamped after this are reported (the
        sampler itself is started before the warm-up so that nvidia-smi is already running)."""
        self.t_mark = datetime.datetime.now()

    def stop(self):
        t_end = datetime.datetime.now()
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        t_mark = getattr(self, "t_mark", None)
        rows = []  # (in the timed window?, sm MHz, max MHz, active reasons)
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                inside = True
                if t_mark is not None:
                    try:
                        ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f")
                        inside = t_mark <= ts <= t_end
                    except ValueError:
                        inside = False
                try:
                    rows.append((inside, float(parts[1]), float(parts[2]),
                                 [nm for nm, v in zip(names, parts[5:9]) if v.lower() == "active"]))
                except ValueError:
                    continue
        os.unlink(self.path)
        timed = [r for r in rows if r[0]]
        window = "timed region"
        if not timed:          # clock skew between nvidia-smi's stamps and ours: keep every sample
            timed, window = rows, "whole run (no sample stamped inside the timed region)"
        sm = [r[1] for r in timed]
        smax = timed[-1][2] if timed else None
        reasons = {nm for r in timed for nm in r[3]}
        loaded = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "window": window}


# ---------------------------------------------------------------------------
# CPU baseline (oracle) — the only place bench.py executes oracle/
# ---------------------------------------------------------------------------

def cpu_nand_sample(seed, gates, threads, exact=False):
    """Time `gates` NANDs on the CPU with `threads` pthreads: the FP64-FFT port
    (default, the fast CPU baseline) or the exact-integer oracle."""
    from oracle import oracle as O

    p = O.default_params()
    keys = O.Keys(p, seed)
    ctx = O.Context(p, keys) if exact else O.FftContext(p, keys)
    rng = np.random.default_rng(seed)
    a = rng.integers(0, 2, gates).astype(np.uint8)
    b = rng.integers(0, 2, gates).astype(np.uint8)
    pool = np.zeros((3 * gates, p.n + 1), np.uint32)
    pool[:gates] = O.encrypt(p, keys, a, seed, 1)
    pool[gates:2 * gates] = O.encrypt(p, keys, b, seed, 2)
    recs = np.zeros(gates, dtype=[("dst", "<u4"), ("src_a", "<u4"), ("src_b", "<u4"), ("src_c", "<u4"),
                                  ("c0", "<u4"), ("alpha", "i1"), ("beta", "i1"), ("kind", "i1"), ("gamma", "i1")])
    c0, al, be = O.GATE_LIN["NAND"]
    recs["dst"] = np.arange(2 * gates, 3 * gates)
    recs["src_a"] = np.arange(gates)
    recs["src_b"] = np.arange(gates, 2 * gates)
    recs["c0"], recs["alpha"], recs["beta"] = c0, al, be

    def step():
        t0 = time.perf_counter()
        ctx.run_gates(recs, pool, threads=threads)
        return time.perf_counter() - t0

    ok = lambda: bool(np.array_equal(O.decrypt(p, keys, pool[2 * gates:]), 1 - (a & b)))  # noqa: E731
    return step, ok


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, dist):
    if dist.rank != 0:
        return None
    threads = os.cpu_count() or 1
    sample = 256 * threads  # ~2 s of wall time per step (~30 core-seconds)
    step, ok = cpu_nand_sample(args.seed, sample, threads)
    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    assert ok(), "CPU FFT port produced wrong NAND outputs"
    value = sample * len(times) / sum(times)
    xstep, xok = cpu_nand_sample(args.seed, 16 * threads, threads, exact=True)
    xdt = xstep()
    assert xok(), "CPU oracle produced wrong NAND outputs"
    line = {
        "impl": "reference",
        "metric": METRIC, "value": value, "unit": "gates/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32 torus; FP64 FFT on the host (bit-exact vs integer oracle)",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "gates_per_step": sample, "sample_of": args.gates},
        "cpu_baseline": {"value": value, "unit": "gates/s", "cores": threads, "kind": "port",
                         "sample": f"{sample} NAND gates per step on {threads} threads ({cpu_model()}); "
                                   "FP64-FFT CPU port oracle/tfhe_cpu_fft.c, 8 gates per SIMD register "
                                   "(reference has no crypto)",
                         "exact_oracle_value": 16 * threads / xdt,
                         "exact_oracle_note": "exact-integer Goldilocks-NTT oracle/tfhe_oracle.c, same threads"},
        "e2e": {"value": value, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    return line


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def bnn_latency(cfg, seed, trials=2, cached=True):
    """BASELINE configs 2-5 through the reference compiler on TfheContext
    (engine created and warmed before the timed flush)."""
    from paper_1806_03461_b200 import workloads
    from paper_1806_03461_b200.backend import TfheContext

    warm = TfheContext(seed=seed)
    warm.decrypt(warm.g_and(warm.encrypt(1), warm.encrypt(1)))  # CUDA context, BK FFT, KSK upload
    # fresh contexts (each builds its DAG from scratch); a second one finds the engine's
    # pools already grown, as a serving process would
    runs = [workloads.run_encrypted(TfheContext, cfg, seed=seed, replays=1, cached=cached and t == trials - 1)
            for t in range(trials)]
    rep = min(runs, key=lambda r: r["first_eval_s"])
    rep["first_eval_trials_s"] = [r["first_eval_s"] for r in runs]
    rep["cached"] = runs[-1]["cached"]
    rep["note"] = ("first_eval_s = encrypt + DAG build through the reference compiler (background device "
                   "flushes overlap it) + final flush + decrypt of one batch, best of the fresh contexts in "
                   "first_eval_trials_s; rates are over first_eval_s; replay.latency_s = a new encrypted "
                   "batch through the same context's DAG (upload, every level on the device, decrypt); "
                   "cached.first_eval_s = a fresh context running the compiled level schedule "
                   "(workloads.compile_schedule) without the reference compiler")
    ref = workloads.run_sim_reference(cfg, seed=seed)
    rep["reference_cpu"] = ref
    rep["counted_gates_match_simcontext"] = ref["counted_gates_per_input"] == rep["counted_gates_per_input"]
    return rep


def bnn_csa_latency(cfg, seed, base):
    """The same config with the opt-in carry-save popcount (TfheContext(csa_popcount=True),
    paper_1806_03461_b200/popcount.py): the reference compiler's popcounts run as
    Wallace-style compressor networks (~2n instead of ~3n bootstraps for n bits); decrypted
    outputs and counted GateStats are the reference's.  `base` = the pure drop-in's report."""
    from paper_1806_03461_b200 import popcount, workloads
    from paper_1806_03461_b200.backend import TfheContext

    class CsaContext(TfheContext):
        def __init__(self, **kw):
            super().__init__(csa_popcount=True, **kw)

    try:
        rep = workloads.run_encrypted(CsaContext, cfg, seed=seed, replays=0 if cfg in ("cfg3", "cfg5") else 1)
    finally:
        popcount.uninstall()
    keep = ("config", "batch", "counted_gates", "counted_gates_per_input", "executed_bootstraps", "levels", "depth",
            "first_eval_s", "dag_build_s", "final_flush_s", "matches_oracle_eval", "replay")
    out = {k: rep[k] for k in keep}
    if isinstance(base, dict) and "executed_bootstraps" in base:
        out["counted_gates_match_simcontext"] = (base.get("counted_gates_match_simcontext") is True
                                                  and base["counted_gates_per_input"] == rep["counted_gates_per_input"]
                                                  and base["depth"] == rep["depth"])
        out["executed_bootstraps_vs_drop_in"] = rep["executed_bootstraps"] / base["executed_bootstraps"]
        out["first_eval_speedup_vs_drop_in"] = base["first_eval_s"] / rep["first_eval_s"]
    return out


def strong_scaling_leg(args, dist, eng, recs, weak_value, weak_ms):
    """cfg1 strong scaling (SURVEY §8e first row): the 4,096 gates of one job
    split over the N ranks (4,096/N per GPU, no collective: gates are
    independent), timed like the weak-scaling steps (L2 flushed, CUDA events on
    the engine stream, max over ranks).  At N = 1 it is the headline step."""
    total = args.gates
    if dist.world == 1:
        return {"gates_total": total, "gates_per_gpu": total, "n_gpus": 1, "value": weak_value,
                "ms_per_step": weak_ms, "unit": "gates/s", "note": "N = 1: identical to the headline step"}
    per = -(-total // dist.world)
    mine = recs[dist.rank * per:min(total, (dist.rank + 1) * per)]
    for _ in range(args.warmup):
        eng.run_gates(mine)
    eng.sync()
    dist.barrier()
    tot = 0.0
    for _ in range(args.steps):
        eng.flush_l2()
        eng.sync()
        eng.run_gates(mine)
        br, ks = eng.last_timing()
        tot += br + ks
    step_s = dist.max(tot / 1e3) / args.steps
    return {"gates_total": total, "gates_per_gpu": per, "n_gpus": dist.world, "value": total / step_s,
            "ms_per_step": 1e3 * step_s, "unit": "gates/s", "scaling": "strong",
            "note": "one 4,096-gate job split over the ranks; time = max over ranks"}


def cggi_layout_leg(args, dist, dev, recs, h_in, steps=5):
    """The same NAND step with the CGGI bootstrapping key (bk_unroll 1: one
    external product per key bit) on a second engine, for comparison with the
    default key-pair layout."""
    from paper_1806_03461_b200 import tfhe

    p = tfhe.default_params()
    p.bk_unroll = 1
    keys = tfhe.KeySet(seed=args.seed, params=p)
    eng = tfhe.Engine(keys, device=dev)
    n = recs.size
    eng.reserve(3 * n)
    eng.upload(0, h_in)
    for _ in range(3):
        eng.run_gates(recs)
    eng.sync()
    dist.barrier()
    tot, brs = 0.0, []
    for _ in range(steps):
        eng.flush_l2()
        eng.sync()
        eng.run_gates(recs)
        br, ks = eng.last_timing()
        brs.append(br)
        tot += br + ks
    value = n * dist.world * steps / dist.max(tot / 1e3)
    eng.close()
    return {"bk_unroll": 1, "value": value, "unit": "gates/s", "blind_rotate_ms": statistics.median(brs),
            "kernel": "k_blind_rotate", "flops_per_bootstrap": F_BS[1], "steps": steps,
            "note": "CGGI key layout (one TGSW per key bit), same inputs, L2 flushed per step"}


def bnn_outp(cfg, seed, dist, dev):
    """N > 1: one batch of BASELINE config `kind` with Out-P:
    every rank evaluates a cost-balanced slice of each layer's output units on
    its own GPU (its own DAG, built concurrently) and the layer's output
    ciphertexts are all-gathered (NCCL) before the next layer.  Time = max over
    ranks from a barrier to the gathered last layer (host DAG build included)."""
    import torch

    from paper_1806_03461_b200 import parallel, workloads
    from paper_1806_03461_b200.backend import TfheContext, shared_keys
    from hebnn.model import oracle_eval

    model, batch = workloads.build(cfg, seed)
    X = workloads.inputs(cfg, model, batch, seed + 1)
    keys = shared_keys(seed)  # deterministic: identical on every rank
    if batch >= dist.world and batch % dist.world == 0:
        return bnn_batch_shards(cfg, model, X, seed, dist, dev)
    cts = keys.encrypt(np.ascontiguousarray(X.T).reshape(-1), seed=seed + 7, stream=900)
    cts = cts.reshape(X.shape[1], batch, -1)
    warm = TfheContext(seed=seed, device=dev)
    warm.decrypt(warm.g_and(warm.encrypt(1), warm.encrypt(1)))
    comm = parallel.TorchComm(device=f"cuda:{dev}" if torch.distributed.get_backend() == "nccl" else "cpu")
    ev = parallel.OutPEvaluator(lambda: TfheContext(seed=seed, device=dev, lanes=batch), comm)
    dist.barrier()
    t0 = time.perf_counter()
    result = ev.run(model, cts)
    elapsed = dist.max(time.perf_counter() - t0)
    rep = {"config": cfg, "batch": batch, "mode": f"Out-P over {dist.world} GPUs", "first_eval_s": elapsed,
           "units_per_rank": [s["units"] for s in ev.stats],
           "executed_bootstraps_this_rank": sum(s["executed"]["bootstraps"] for s in ev.stats)}
    if dist.rank == 0:
        ctx = TfheContext(seed=seed, device=dev, lanes=batch)
        if model.output_mode == "score_words":
            got = parallel.decode_scores(ctx, result)
        else:
            bits = keys.decrypt(np.stack(result).reshape(-1, cts.shape[-1])).reshape(len(result), batch)
            got = np.where(bits.T == 1, 1, -1)
        rep["matches_oracle_eval"] = all(list(got[b]) == oracle_eval(model, [1 if v else -1 for v in X[b]])
                                         for b in range(batch))
    return rep


def bnn_batch_shards(cfg, model, X, seed, dist, dev):
    """Batched configs (cfg3/cfg4 batch 8, cfg5 batch 64 "sharded across 8
    GPUs"): the records are split evenly over the ranks, each rank evaluates
    its shard as lanes of one DAG on its GPU; time = max over ranks."""
    from paper_1806_03461_b200 import workloads
    from paper_1806_03461_b200.backend import TfheContext
    from hebnn.compiler import eval_model
    from hebnn.model import oracle_eval

    per = X.shape[0] // dist.world
    mine = X[dist.rank * per:(dist.rank + 1) * per]
    warm = TfheContext(seed=seed, device=dev)
    warm.decrypt(warm.g_and(warm.encrypt(1), warm.encrypt(1)))
    dist.barrier()
    t0 = time.perf_counter()
    ctx = TfheContext(seed=seed, device=dev, lanes=per, enc_stream=700 + dist.rank)
    outs, _ = eval_model(ctx, model, ctx.encrypt_many(mine.T))
    got = workloads.decode_outputs(ctx, outs)
    elapsed = dist.max(time.perf_counter() - t0)
    ok = all(list(got[b]) == oracle_eval(model, [1 if v else -1 for v in mine[b]]) for b in range(per))
    ok = dist.max(0.0 if ok else 1.0) == 0.0
    return {"config": cfg, "batch": X.shape[0], "mode": f"batch sharded over {dist.world} GPUs ({per} per GPU)",
            "first_eval_s": elapsed, "records_per_s": X.shape[0] / elapsed, "matches_oracle_eval": ok,
            "executed_bootstraps_this_rank": ctx.exec_stats["bootstraps"]}


def last_profiled_traffic(kernel="k_blind_rotate"):
    """DRAM bytes per launch of `kernel` from the newest profiles/*/traffic.json
    (written by scripts/ncu_summary.py from an `ncu --set full` capture)."""
    base = os.path.join(ROOT, "profiles")
    best = None
    def natural(name):  # r01_v11 after r01_v8
        return [int(t) if t.isdigit() else t for t in re.split(r"(\d+)", name)]

    for d in sorted(os.listdir(base), key=natural) if os.path.isdir(base) else []:
        f = os.path.join(base, d, "traffic.json")
        if os.path.exists(f):
            best = f
    if not best:
        return None, None
    with open(best) as fh:
        data = json.load(fh)
    return data.get("dram_bytes_per_launch", {}).get(kernel), os.path.relpath(os.path.dirname(best), ROOT)


def run_ours(args, dist):
    import torch

    from paper_1806_03461_b200 import tfhe

    if args.plan:
        ranks = dist.gather_obj({"rank": dist.rank, "local_rank": dist.local_rank,
                                 "world": dist.world, "pid": os.getpid()})
        return {"plan": True, "n_gpus": dist.world, "backend": dist.backend, "ranks": ranks,
                "share_gpu": dist.share}
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the engine has no CPU fallback)")
    dev = dist.local_rank
    keys = tfhe.KeySet(seed=args.seed)
    from paper_1806_03461_b200 import backend as _backend
    _backend._KEY_CACHE.setdefault(args.seed, keys)  # the BNN leg's contexts reuse these keys
    eng = tfhe.Engine(keys, device=dev)
    n = args.gates
    rng = np.random.default_rng(1000 + dist.rank)
    a = rng.integers(0, 2, n).astype(np.uint8)
    b = rng.integers(0, 2, n).astype(np.uint8)
    words = keys.params.n + 1
    # pinned host staging (torch is plumbing here)
    h_in = torch.empty((2 * n, words), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    h_in[:n] = keys.encrypt(a, seed=args.seed, stream=2 * dist.rank + 1)
    h_in[n:] = keys.encrypt(b, seed=args.seed, stream=2 * dist.rank + 2)
    h_out = torch.empty((n, words), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    eng.reserve(3 * n)
    eng.upload(0, h_in)
    recs = tfhe.gate_records(n)
    c0, al, be = tfhe.GATE_LIN["NAND"]
    recs["dst"] = np.arange(2 * n, 3 * n)
    recs["src_a"] = np.arange(n)
    recs["src_b"] = np.arange(n, 2 * n)
    recs["c0"], recs["alpha"], recs["beta"] = c0, al, be

    fp64_peak = eng.measure_fp64_peak()

    clocks = ClockSampler(dev)
    clocks.start()               # before the warm-up: nvidia-smi needs ~0.3 s to come up
    for _ in range(args.warmup):
        eng.run_gates(recs)
        eng.sync()
    eng.sync()
    dist.barrier()
    launches0 = eng.counters()["kernel_launches"]
    clocks.mark()                # samples from here to stop() are the timed region's
    step_ms, br_ms, ks_ms = [], [], []
    for _ in range(args.steps):
        eng.flush_l2()           # cold L2 for every timed step
        eng.sync()
        eng.run_gates(recs)
        br, ks = eng.last_timing()  # CUDA events on the engine stream
        br_ms.append(br)
        ks_ms.append(ks)
        step_ms.append(br + ks)
    eng.sync()
    clk = clocks.stop()
    launches = eng.counters()["kernel_launches"] - launches0
    out = eng.download(2 * n, n)
    correct = bool(np.array_equal(keys.decrypt(out), 1 - (a & b)))

    total_s = dist.max(sum(step_ms) / 1e3)
    value = n * dist.world * args.steps / total_s

    # e2e through the C ABI with host buffers: every step uploads its inputs from
    # pinned memory and downloads its outputs; the copies run on the engine's
    # copy streams, overlapping the neighbouring steps' compute (two slot
    # regions, double-buffered host staging)
    dist.barrier()
    eng.reserve(6 * n)
    h_in2 = [h_in, torch.empty((2 * n, words), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)]
    h_in2[1][:] = h_in
    h_out2 = [h_out, torch.empty((n, words), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)]
    recs2 = [recs, recs.copy()]
    for f in ("dst", "src_a", "src_b"):
        recs2[1][f] = recs[f] + 3 * n
    eng.sync()
    t0 = time.perf_counter()
    for k in range(args.steps):
        r = k % 2
        eng.upload_async(3 * n * r, h_in2[r])
        eng.run_gates(recs2[r])
        eng.download_async(3 * n * r + 2 * n, h_out2[r])
    eng.sync()
    e2e_total = dist.max(time.perf_counter() - t0)
    e2e_value = n * dist.world * args.steps / e2e_total
    # the same without overlap: blocking upload -> gates -> blocking download per step
    dist.barrier()
    t0 = time.perf_counter()
    for k in range(args.steps):
        eng.upload(0, h_in)
        eng.run_gates(recs)
        eng.download(2 * n, n, out=h_out)
    e2e_serial = n * dist.world * args.steps / dist.max(time.perf_counter() - t0)
    correct &= bool(np.array_equal(keys.decrypt(h_out), 1 - (a & b)))
    correct &= bool(np.array_equal(keys.decrypt(h_out2[0]), 1 - (a & b)))
    correct &= bool(np.array_equal(keys.decrypt(h_out2[1]), 1 - (a & b))) or args.steps < 2

    br_med = statistics.median(br_ms)
    unroll = 2 if keys.params.bk_unroll == 2 else 1
    # roofline.achieved uses SURVEY.md §8(d)'s fixed per-bootstrap figure (F_BS1, the
    # CGGI blind rotation), whatever the blind-rotation algorithm; the key-pair
    # algorithm executes F_BS2 flops, reported beside it as achieved_executed
    achieved = n * F_BS1 / (br_med / 1e3) / 1e12
    achieved_exec = n * F_BS[unroll] / (br_med / 1e3) / 1e12
    traffic, traffic_src = last_profiled_traffic()
    # nominal FP64 peak: 64 DFMA lanes per SM x 2 flops x max SM clock
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    nominal = sms * 128 * clk["sm_max_mhz"] * 1e6 / 1e12 if clk.get("sm_max_mhz") else None
    line = {
        "metric": METRIC, "value": value, "unit": "gates/s", "n_gpus": dist.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dist.max(statistics.mean(step_ms)), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "u32 torus; FP64 negacyclic FFT (bit-exact vs integer oracle)", "data": "synthetic",
        "config": {"workload": WORKLOAD, "gates_per_gpu": n, "parallelism": f"replicated keys, {dist.world} GPU(s)",
                   "l2": "flushed (256 MiB write) before every timed step", "inputs": "resident in HBM"},
        "e2e": {"value": e2e_value, "unit": "gates/s", "h2d_bytes_per_step": int(h_in.nbytes + recs.nbytes),
                "d2h_bytes_per_step": int(h_out.nbytes),
                "serial_value": e2e_serial,
                "note": "C ABI, pinned host buffers, H2D/D2H on copy streams overlapping neighbouring steps; "
                        "serial_value: blocking copies, no overlap"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp64_peak, "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": "k_blind_rotate_u2" if unroll == 2 else "k_blind_rotate",
                     "flops_per_bootstrap": F_BS1,
                     "flops_per_bootstrap_note": "SURVEY.md 8(d) fixed figure (CGGI blind rotation: 630 external "
                                                 "products); the key-pair blind rotation run here executes "
                                                 f"{F_BS[unroll]} FP64 flops",
                     "achieved_executed": achieved_exec, "frac_executed": achieved_exec / fp64_peak,
                     "peak_source": "DFMA micro-benchmark in this run (MEASURED_PEAKS.json has no FP64 figure)",
                     "peak_nominal": nominal, "frac_of_nominal": (achieved / nominal) if nominal else None},
        "kernel_ms": {"blind_rotate": br_med, "key_switch": statistics.median(ks_ms)},
        "clocks": clk,
        "correct": correct,
    }
    line["strong_scaling"] = strong_scaling_leg(args, dist, eng, recs, value, statistics.mean(step_ms))
    if not args.no_compare:
        line["alt_layout"] = cggi_layout_leg(args, dist, dev, recs, h_in)
    if args.bnn_list:
        line["bnn"] = {}
    for cfg in args.bnn_list:
        try:
            if dist.world > 1:
                rep = bnn_outp(cfg, args.seed, dist, dev)
            elif dist.rank == 0:
                # the two largest configs skip the cached leg (same device work as their replay;
                # tests/test_gpu_reference_replay.py runs it) to keep the default run in minutes
                rep = bnn_latency(cfg, args.seed, trials=2 if cfg in ("cfg2n", "cfg2l") else 1,
                                  cached=cfg not in ("cfg3", "cfg5"))
            else:
                rep = None
        except Exception as exc:  # report, never hide
            rep = {"error": repr(exc)}
        if dist.rank == 0:
            line["bnn"][cfg] = rep
        if dist.rank == 0 and dist.world == 1 and not args.no_csa:
            try:
                line.setdefault("bnn_csa", {})[cfg] = bnn_csa_latency(cfg, args.seed, rep)
            except Exception as exc:  # report, never hide
                line.setdefault("bnn_csa", {})[cfg] = {"error": repr(exc)}
        if dist.world > 1 and not args.no_csa:
            # the same Out-P / batch-sharded evaluation with the carry-save popcount on every rank
            # (TfheContext reads the default of csa_popcount from the environment)
            os.environ["HEBNN_B200_CSA_POPCOUNT"] = "1"
            try:
                rep_csa = bnn_outp(cfg, args.seed, dist, dev)
            except Exception as exc:  # report, never hide
                rep_csa = {"error": repr(exc)}
            finally:
                os.environ.pop("HEBNN_B200_CSA_POPCOUNT", None)
                from paper_1806_03461_b200 import popcount

                popcount.uninstall()
            if dist.rank == 0:
                line.setdefault("bnn_csa", {})[cfg] = rep_csa
    if args.bnn_list and dist.rank == 0 and dist.world == 1:
        try:  # the shipped Cancer model on the reference dataset's 569 rows, as lanes (f4)
            from paper_1806_03461_b200 import workloads
            from paper_1806_03461_b200.backend import TfheContext

            rep = workloads.run_cancer(TfheContext, seed=args.seed)
            rep.pop("predictions")
            line["cancer"] = rep
        except Exception as exc:  # report, never hide
            line["cancer"] = {"error": repr(exc)}
        if not args.no_csa:
            try:  # the same rows with the opt-in carry-save popcount
                from paper_1806_03461_b200 import popcount

                class CsaContext(TfheContext):
                    def __init__(self, **kw):
                        super().__init__(csa_popcount=True, **kw)

                try:
                    rep = workloads.run_cancer(CsaContext, seed=args.seed)
                finally:
                    popcount.uninstall()
                rep.pop("predictions")
                line["cancer_csa"] = rep
            except Exception as exc:  # report, never hide
                line["cancer_csa"] = {"error": repr(exc)}
    if args.bnn_list and dist.rank == 0 and dist.world == 1:
        # first-evaluation latency per config at a glance (details in bnn / bnn_csa)
        line["bnn_first_eval_s"] = {
            cfg: {"drop_in": (line["bnn"].get(cfg) or {}).get("first_eval_s"),
                  "csa_popcount": (line.get("bnn_csa", {}).get(cfg) or {}).get("first_eval_s")}
            for cfg in args.bnn_list}
    if args.bnn_list and dist.rank == 0:
        line["bnn_all_match_oracle_eval"] = all(
            isinstance(r, dict) and r.get("matches_oracle_eval") is True
            and (r.get("replay") or {}).get("matches_oracle_eval", True) is True
            and (r.get("cached") or {}).get("matches_oracle_eval", True) is True
            for r in list(line["bnn"].values()) + list(line.get("bnn_csa", {}).values()))
    if dist.world > 1:
        dist.barrier()
        lines = dist.nccl_lines()
        if dist.rank == 0:
            line["nccl"] = {"backend": dist.backend, "log_lines": lines}
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        sample = 512 * threads  # ~5 s of wall time (~80 core-seconds) of FP64-FFT CGGI on the host
        step, ok = cpu_nand_sample(args.seed, sample, threads)
        step()  # warm the caches and the threads
        dt = step()
        line["cpu_baseline"] = {"value": sample / dt, "unit": "gates/s", "cores": threads, "kind": "port",
                                "sample": f"{sample} NAND gates on {threads} threads ({cpu_model()}), "
                                          f"{dt:.1f} s; FP64-FFT CPU port oracle/tfhe_cpu_fft.c, 8 gates per SIMD "
                                          "register, bit-exact vs the integer oracle (reference has no crypto)",
                                "correct": ok()}
        step1, _ = cpu_nand_sample(args.seed + 1, 64, 1)
        line["cpu_baseline"]["single_thread_value"] = 64 / step1()
        xstep, xok = cpu_nand_sample(args.seed, 16 * threads, threads, exact=True)
        xdt = xstep()
        line["cpu_baseline"]["exact_oracle_value"] = 16 * threads / xdt
        line["cpu_baseline"]["exact_oracle_note"] = ("exact-integer Goldilocks-NTT oracle/tfhe_oracle.c, "
                                                     f"{16 * threads} gates on {threads} threads; correct={xok()}")
    eng.close()
    return line


def main():
    args = parse_args()
    world = os.environ.get("WORLD_SIZE")
    if args.impl == "ours" and args.gpus > 1 and world is None:
        sys.exit(spawn_ranks(args))
    if args.impl == "ours" and world is not None and int(world) != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}: refusing to report a wrong n_gpus")
    if args.impl == "reference":
        # CPU arm: rank 0 alone runs; no process group, other ranks exit 0 without work
        if int(os.environ.get("RANK", "0")) != 0:
            return
        line = run_reference(args, _Rank0())
        print(json.dumps(line), flush=True)
        return
    dist = Dist()
    try:
        line = run_reference(args, dist) if args.impl == "reference" else run_ours(args, dist)
        if dist.rank == 0 and line is not None:
            print(json.dumps(line), flush=True)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
