#!/bin/bash
# HMMA low-rank kernel: 16-entry stages (3) vs 8-entry stages (7), x ring producer warps
set -u
mkdir -p gpurun_out
for r in 1 2; do
  for spec in 16:2 16:3 8:2 8:3; do
    eps=${spec%%:*}; np=${spec#*:}
    PIKV_BF16TC_EPS=$eps PIKV_RING_PROD=$np python bench.py --config c4-lowrank --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bx_${eps}_${np}_$r.json 2> /dev/null
    python - "gpurun_out/bx_${eps}_${np}_$r.json" "$eps" "$np" <<'PY'
import json, sys
f, e, np_ = sys.argv[1:4]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print("eps %2s prod %s %9.0f tok/s %7.4f ms  attend %.4f ms frac %.3f share %.3f  e2e %9.0f" % (e, np_, d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["roofline"]["attend_share_of_step"], d["e2e"]["value"]))
except Exception as ex:
    print(e, np_, "failed", ex)
PY
  done
done
