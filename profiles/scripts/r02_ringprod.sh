#!/bin/bash
# tensor-core attention rings: two producer warps (default with static shares) vs one (PIKV_RING_PROD=1)
set -u
mkdir -p gpurun_out
for r in 1 2; do
  for spec in c4-lowrank:2 c4-lowrank:1 c4-int4:2 c4-int4:1; do
    c=${spec%%:*}; np=${spec#*:}
    if [ $np = 1 ]; then export PIKV_RING_PROD=1; else unset PIKV_RING_PROD; fi
    python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/rp_${c}_${np}_$r.json 2> /dev/null
    python - "gpurun_out/rp_${c}_${np}_$r.json" "$c" "$np" <<'PY'
import json, sys
f, c, np_ = sys.argv[1:4]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print("%-11s prod %s %9.0f tok/s %7.4f ms  attend %.4f ms frac %.3f share %.3f  e2e %9.0f" % (c, np_, d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["roofline"]["attend_share_of_step"], d["e2e"]["value"]))
except Exception as ex:
    print(c, np_, "failed", ex)
PY
  done
done
