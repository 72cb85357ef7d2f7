#!/bin/bash
# micro-batches per step (2 vs 4) with static shares (run on the GPU box)
set -u
mkdir -p gpurun_out
for r in 1 2; do
  for c in c4-lowrank c4-int4 c5 c4-int8 c2; do
    for mb in 2 4; do
      python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --micro $mb > gpurun_out/mb_${c}_${mb}_$r.json 2> /dev/null
      python - "gpurun_out/mb_${c}_${mb}_$r.json" "$c" "$mb" <<'PY'
import json, sys
f, c, mb = sys.argv[1:4]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print("%-11s micro %s %9.0f tok/s %7.4f ms  attend %.4f ms frac %.3f share %.3f  e2e %9.0f" % (c, mb, d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["roofline"]["attend_share_of_step"], d["e2e"]["value"]))
except Exception as ex:
    print(c, mb, "failed", ex)
PY
    done
  done
done
