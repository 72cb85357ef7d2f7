#!/bin/bash
# tensor-core attention configs (static shares, two ring producers): attention SMs sweep
set -u
mkdir -p gpurun_out
for r in 1 2; do
  for spec in c4-int4:108 c4-int4:116 c4-int4:124 c4-int4:132 c4-lowrank:108 c4-lowrank:116 c4-lowrank:124; do
    c=${spec%%:*}; sms=${spec#*:}
    python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --attend-sms $sms > gpurun_out/ts_${c}_${sms}_$r.json 2> /dev/null
    python - "gpurun_out/ts_${c}_${sms}_$r.json" "$c" "$sms" <<'PY'
import json, sys
f, c, sms = sys.argv[1:4]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print("%-11s sms %4s %9.0f tok/s %7.4f ms  attend %.4f ms frac %.3f share %.3f  e2e %9.0f" % (c, sms, d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["roofline"]["attend_share_of_step"], d["e2e"]["value"]))
except Exception as ex:
    print(c, sms, "failed", ex)
PY
  done
done
