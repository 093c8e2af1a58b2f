#!/bin/bash
# time experimental library variants (gpu_timing: 4096 NANDs); correctness not expected for skip variants
for lib in paper_1806_03461_b200/_lib/libhebnn_b200.so paper_1806_03461_b200/_lib/exp_*.so; do
  echo "== $lib"; HEBNN_B200_LIB=$PWD/$lib timeout 120 python scripts/gpu_timing.py 2>&1 | tail -2 | head -1
done
