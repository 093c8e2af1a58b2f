#!/bin/bash
# Usage: scripts/profile_round.sh <tag>   (run under gpurun; results in gpurun_out/<tag>/)
# bench line, ncu launch list of the bench step, ncu --set full of the dominant kernels
# (blind rotation, key switch) and of the lone-level 8-CTA bin-split kernel.
set -u
TAG=${1:-prof}
OUT=gpurun_out/$TAG
mkdir -p $OUT
CMD="python bench.py --steps 3 --warmup 3 --bnn none --no-cpu-baseline --no-compare"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi.txt 2>&1
$CMD > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
$CMD > $OUT/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_blind_rotate -s 3 -c 1 -o $OUT/k_blind_rotate $CMD > $OUT/ncu_br.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_keyswitch -s 3 -c 1 -o $OUT/k_keyswitch $CMD > $OUT/ncu_ks.log 2>&1
python scripts/narrow_levels.py 1 > $OUT/binsplit_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_blind_rotate_u2_binsplit -s 2 -c 1 -o $OUT/k_binsplit python scripts/narrow_levels.py 1 > $OUT/ncu_binsplit.log 2>&1
ls -la $OUT
