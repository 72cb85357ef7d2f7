#!/bin/bash
# micro-batch pipeline: cross-micro-batch attention ordering by stream event (gate 0)
# vs the progress gate (PIKV_GROUP_GATE = percent of the previous attention's CTAs done)
set -u
mkdir -p gpurun_out
for r in 1 2; do
  for c in ${1:-c2 c4-lowrank c5}; do
    for gt in 0 50 80 95; do
      PIKV_GROUP_GATE=$gt python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/gt_${c}_${gt}_$r.json 2> /dev/null
      python - "gpurun_out/gt_${c}_${gt}_$r.json" "$c" "$gt" <<'PY'
import json, sys
f, c, gt = sys.argv[1:4]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print("%-11s gate %3s %9.0f tok/s %7.4f ms  attend %.4f ms frac %.3f share %.3f  e2e %9.0f" % (c, gt, d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["roofline"]["attend_share_of_step"], d["e2e"]["value"]))
except Exception as ex:
    print(c, gt, "failed", ex)
PY
    done
  done
done
