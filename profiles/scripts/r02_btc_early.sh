#!/bin/bash
# HMMA low-rank kernel: stage released after the fragment loads (default) vs after the math
# (PIKV_BF16TC_LATE=1), x attention SMs (run on the GPU box)
set -u
mkdir -p gpurun_out
for r in 1 2; do
  for spec in early:116 late:116 early:124 early:132; do
    k=${spec%%:*}; sms=${spec#*:}
    if [ $k = late ]; then export PIKV_BF16TC_LATE=1; else unset PIKV_BF16TC_LATE; fi
    python bench.py --config c4-lowrank --steps 50 --warmup 5 --no-cpu-baseline --attend-sms $sms > gpurun_out/be_${k}_${sms}_$r.json 2> /dev/null
    python - "gpurun_out/be_${k}_${sms}_$r.json" "$k" "$sms" <<'PY'
import json, sys
f, k, sms = sys.argv[1:4]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print("%-5s sms %4s %9.0f tok/s %7.4f ms  attend %.4f ms frac %.3f share %.3f  e2e %9.0f" % (k, sms, d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["roofline"]["attend_share_of_step"], d["e2e"]["value"]))
except Exception as ex:
    print(k, sms, "failed", ex)
PY
  done
done
