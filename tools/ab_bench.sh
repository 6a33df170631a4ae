#!/bin/bash
# A/B timing of library variants (run under gpurun): for each .so given, copy it over liblocc.so and run
# the C3 bench with the encoder trace summary.  usage: tools/ab_bench.sh variant.so ...
set -e
cp paper_2304_09439_b200/liblocc.so /tmp/liblocc_base.so
for so in /tmp/liblocc_base.so "$@"; do
  cp "$so" paper_2304_09439_b200/liblocc.so; touch paper_2304_09439_b200/liblocc.so
  echo "== $so"
  python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-grad --no-cells --no-sim --no-sweep \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value']), 'enc ms', round(d['roofline']['avg_launch_ms'],2), 'frac', round(d['roofline']['frac'],3))"
  python tools/trace_run.py > /tmp/tr.txt 2>&1 && python tools/trace_summary.py /tmp/tr.txt 2>/dev/null | head -3 || true
done
cp /tmp/liblocc_base.so paper_2304_09439_b200/liblocc.so; touch paper_2304_09439_b200/liblocc.so
