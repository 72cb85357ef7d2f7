#!/bin/bash
# micro-batch pipeline: attention ordered by stream events on all SMs (green 0) vs each
# micro-batch's attention in a green-context SM partition without ordering (PIKV_GREEN=1)
set -u
mkdir -p gpurun_out
for r in 1 2; do
  for c in ${1:-c2 c3 c4-lowrank c4-int4 c5}; do
    for gr in 0 1; do
      PIKV_GREEN=$gr python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/gr_${c}_${gr}_$r.json 2> gpurun_out/gr_${c}_${gr}_$r.err
      python - "gpurun_out/gr_${c}_${gr}_$r.json" "$c" "$gr" <<'PY'
import json, sys
f, c, gr = sys.argv[1:4]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print("%-11s green %s %9.0f tok/s %7.4f ms  attend %.4f ms frac %.3f share %.3f  e2e %9.0f" % (c, gr, d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["roofline"]["attend_share_of_step"], d["e2e"]["value"]))
except Exception as ex:
    print(c, gr, "failed", ex)
PY
    done
  done
done
