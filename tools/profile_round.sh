#!/bin/bash
# Round profile (run under gpurun, 1 GPU): plain bench, ncu launch list of one step, ncu --set full
# of each hot kernel.  Usage: tools/profile_round.sh <tag> [pairs]
set -e
TAG=${1:-r1}; PAIRS=${2:-262144}
CMD="python bench.py --pairs $PAIRS --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-grad --no-cells --no-sim --no-sweep"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1
# launch list: skip shape prep (2 launches) + the warm-up step (7 per sub-batch); capture one step
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    -s 2 -c 40 $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
for K in encoder_tc crop_compact head_tc; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/prof_${TAG}_$K $CMD \
      > gpurun_out/ncu_${TAG}_$K.log 2>&1 || true
  ncu -i gpurun_out/prof_${TAG}_$K.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_$K.csv 2>/dev/null || true
  ncu -i gpurun_out/prof_${TAG}_$K.ncu-rep --page details > gpurun_out/details_${TAG}_$K.txt 2>/dev/null || true
done
