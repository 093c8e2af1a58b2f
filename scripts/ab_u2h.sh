#!/bin/bash
# A/B of the wide-level key-pair kernel: 128 threads per bootstrap (u2h) vs 64 (u2)
OUT=${1:-gpurun_out/ab}
mkdir -p $OUT
for v in 1 0; do
  HEBNN_B200_U2H=$v python bench.py --steps 10 --warmup 3 --bnn none --no-cpu-baseline --no-compare > $OUT/bench_u2h$v.json 2> $OUT/bench_u2h$v.err
  python -c "import json,sys; d=json.load(open('$OUT/bench_u2h$v.json')); print('u2h=$v', round(d['value']), d['kernel_ms'], round(d['roofline']['frac_executed'],3), d['correct'])"
done
