"""Summarise ncu reports into profiles/<tag>/: key metrics per kernel + the launch-list shares.
Usage: python scripts/ncu_summary.py gpurun_out/<tag> profiles/<tag>"""
import csv
import io
import os
import subprocess
import sys
from collections import defaultdict

src, dst = sys.argv[1], sys.argv[2]
os.makedirs(dst, exist_ok=True)
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__shared_mem_per_block_static", "launch__grid_size",
    "launch__block_size", "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
]
lines = []
traffic = {}
for rep in sorted(f for f in os.listdir(src) if f.endswith(".ncu-rep")):
    out = subprocess.run(["ncu", "-i", os.path.join(src, rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        continue
    h, units, v = rows[0], rows[1], rows[2]
    lines.append(f"## {rep}  ({v[h.index('Kernel Name')][:80]})")
    for k in KEYS:
        if k in h:
            i = h.index(k)
            lines.append(f"- {k}: {v[i]} {units[i]}")
    lines.append("")
    if "dram__bytes_read.sum" in h:
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(v[h.index("dram__bytes_read.sum")]) * mult.get(units[h.index("dram__bytes_read.sum")], 1)
        wr = float(v[h.index("dram__bytes_write.sum")]) * mult.get(units[h.index("dram__bytes_write.sum")], 1)
        traffic[rep.replace(".ncu-rep", "")] = rd + wr
        tmult = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}
        ti = h.index("gpu__time_duration.sum")
        dur = float(v[ti]) * tmult.get(units[ti], 1e-3)
        try:  # driver-written, per pod
            import json
            hbm = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                              "MEASURED_PEAKS.json")))["hbm_gbs"]
        except (OSError, KeyError, ValueError):
            hbm = 6547.5  # B200_PROFILING.md fallback
        lines.insert(-1, f"- DRAM bandwidth: {(rd + wr) / dur / 1e9:.1f} GB/s = {100 * (rd + wr) / dur / 1e9 / hbm:.2f}% "
                         f"of the measured {hbm} GB/s")
launch = os.path.join(src, "launches.csv")
if os.path.exists(launch):
    txt = [l for l in open(launch) if not l.startswith("==")]
    rows = list(csv.reader(txt))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[1:]:
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        agg[r[ki].split("(")[0][-40:]].append(float(r[vi].replace(",", "")) * scale)
    tot = sum(sum(v) for v in agg.values())
    lines.append("## launch list (ncu gpu__time_duration, cold-cache, serialised)")
    for k, vals in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"- {k}: {len(vals)} launches, mean {sum(vals)/len(vals):.1f} us, share {100*sum(vals)/tot:.1f}%")
import json
json.dump({"dram_bytes_per_launch": traffic, "source": dst}, open(os.path.join(dst, "traffic.json"), "w"), indent=1)
open(os.path.join(dst, "ncu_summary.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
