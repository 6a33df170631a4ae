#!/bin/bash
# Profile the encoder on a B200 (run under gpurun).  Usage: tools/profile_tc.sh <tag> [pairs] [precision] [kernel-regex]
set -e
TAG=${1:-r1}; PAIRS=${2:-16384}; PREC=${3:-bf16}; KRE=${4:-encoder}
CMD="python bench.py --pairs $PAIRS --precision $PREC --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:$KRE -s 1 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv
ncu -i gpurun_out/prof_$TAG.ncu-rep --page details > gpurun_out/details_$TAG.txt
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv > gpurun_out/source_$TAG.csv 2>/dev/null || true
