"""`hebnn` CLI on the B200 engine.

    python -m paper_1806_03461_b200.cli [--backend tfhe-b200|sim] [--key-seed S] [--device D] \
        eval|estimate|fold|ternarize|selftest ...  (the reference's sub-commands and flags)
    python -m paper_1806_03461_b200.cli calibrate    # measured B200 cost-model constants

The reference CLI hard-wires `SimContext()` (cli.py:72, 91, 214-218); this
wrapper rebinds that name to `TfheContext`, so `eval` runs the real encrypted
evaluation on the GPU with the reference's own argument parsing, outputs and
exit codes (cli.py:273-279).  `--t-gate b200` replaces the paper's
t_gate = 0.1 s (costs.py:26) by the measured per-wave bootstrap latency and
sets `--intra-workers` to the bootstraps one B200 keeps in flight, so
`estimate`'s out_seq/out_16p/out_full_p describe B200s.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np


def calibrate(device=0, gates=None, seed=1):
    """Measure one full wave of independent NANDs: returns (t_gate seconds per
    wave, concurrent bootstraps per GPU)."""
    from . import tfhe

    keys = tfhe.KeySet(seed=seed)
    eng = tfhe.Engine(keys, device=device)
    try:
        import torch

        sms = torch.cuda.get_device_properties(device).multi_processor_count
    except Exception:  # pragma: no cover
        sms = 148
    workers = 4 * sms  # k_blind_rotate: 4 bootstraps per SM
    n = gates or workers
    rng = np.random.default_rng(seed)
    cts = keys.encrypt(rng.integers(0, 2, 2 * n).astype(np.uint8), seed=seed, stream=1)
    eng.reserve(3 * n)
    eng.upload(0, cts)
    recs = tfhe.gate_records(n)
    c0, al, be = tfhe.GATE_LIN["NAND"]
    recs["dst"], recs["src_a"], recs["src_b"] = np.arange(2 * n, 3 * n), np.arange(n), np.arange(n, 2 * n)
    recs["c0"], recs["alpha"], recs["beta"] = c0, al, be
    eng.run_gates(recs)
    eng.sync()
    times = []
    for _ in range(3):
        eng.run_gates(recs)
        br, ks = eng.last_timing()
        times.append((br + ks) / 1e3)
    eng.close()
    waves = -(-n // workers)
    return min(times) / waves, workers


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    pre = argparse.ArgumentParser(add_help=False)
    pre.add_argument("--backend", choices=("tfhe-b200", "sim"), default="tfhe-b200")
    pre.add_argument("--key-seed", type=int, default=0)
    pre.add_argument("--device", type=int, default=0)
    pre.add_argument("--csa-popcount", action="store_true",
                     help="popcounts as carry-save compressor networks (popcount.py): ~40%% fewer bootstraps, "
                          "same outputs and counted gates")
    known, rest = pre.parse_known_args(argv)

    if rest[:1] == ["calibrate"]:
        t_gate, workers = calibrate(known.device)
        print(json.dumps({"t_gate_s": t_gate, "intra_workers": workers,
                          "note": "per-wave latency of independent bootstrapped gates on one B200"}))
        return 0

    if "--t-gate" in rest:
        i = rest.index("--t-gate")
        if i + 1 < len(rest) and rest[i + 1] == "b200":
            t_gate, workers = calibrate(known.device)
            rest[i + 1] = repr(t_gate)
            if "--intra-workers" not in rest:
                rest += ["--intra-workers", str(workers)]

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ref = os.path.join(root, "baseline", "_ref")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import hebnn.cli as ref_cli

    if known.backend == "tfhe-b200":
        from .backend import TfheContext

        seed, device, csa = known.key_seed, known.device, (True if known.csa_popcount else None)
        ref_cli.SimContext = lambda: TfheContext(seed=seed, device=device, csa_popcount=csa)
    t0 = time.perf_counter()
    rc = ref_cli.main(rest)
    print(f"[hebnn-b200] backend={known.backend} wall={time.perf_counter() - t0:.3f}s", file=sys.stderr)
    return rc


if __name__ == "__main__":
    sys.exit(main())
