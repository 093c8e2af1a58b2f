"""Aggregate ncu warp-stall samples by CUDA source line (and by phase tag).

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > mix.csv
    python scripts/ncu_source_stalls.py mix.csv [top_n]

Prints the source lines with the most stall samples, each with its dominant
stall reasons and executed warp instructions.
"""

import csv
import collections
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file, cur_line, cur_src = "?", 0, ""
samples = collections.Counter()
inst = collections.Counter()
reasons = collections.defaultdict(collections.Counter)
src_text = {}
header = None
total = 0
with open(path, newline="") as f:
    for row in csv.reader(f):
        if not row:
            continue
        if row[0] == "File Path":
            cur_file = row[1].rsplit("/", 1)[-1]
            continue
        if row[0] == "Line No":
            header = row
            continue
        if header is None or len(row) < len(header):
            continue
        if row[0] not in ("",):
            cur_line, cur_src = int(row[0]), row[1]
            src_text[(cur_file, cur_line)] = cur_src.strip()
        if row[2] in ("", "...") or not row[2].startswith("0x"):
            continue
        rec = dict(zip(header[2:], row[2:]))
        try:
            s = int(rec["Warp Stall Sampling (All Samples)"])
        except (KeyError, ValueError):
            continue
        key = (cur_file, cur_line)
        samples[key] += s
        total += s
        try:
            inst[key] += int(rec["Instructions Executed"])
        except ValueError:
            pass
        for h in header[2:]:
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    v = int(rec[h])
                except ValueError:
                    continue
                if v:
                    reasons[key][h[6:]] += v
print(f"total samples {total}")
for key, s in samples.most_common(top):
    r = ", ".join(f"{k} {v * 100 / s:.0f}%" for k, v in reasons[key].most_common(4))
    print(f"{s * 100 / total:5.1f}%  {key[0]}:{key[1]:<4d} inst {inst[key] / 1e6:8.1f}M  [{r}]  {src_text.get(key, '')[:90]}")
