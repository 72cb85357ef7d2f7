#!/bin/bash
# c2 / c3 with static shares: attention SMs sweep (run on the GPU box)
set -u
mkdir -p gpurun_out
for r in 1 2; do
  for c in c2 c3; do
    for sms in 104 112 116 120 124; do
      python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --attend-sms $sms > gpurun_out/cs_${c}_${sms}_$r.json 2> /dev/null
      python - "gpurun_out/cs_${c}_${sms}_$r.json" "$c" "$sms" <<'PY'
import json, sys
f, c, sms = sys.argv[1:4]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print("%-4s sms %4s %9.0f tok/s %7.4f ms  attend %.4f ms frac %.3f share %.3f  e2e %9.0f" % (c, sms, d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["roofline"]["attend_share_of_step"], d["e2e"]["value"]))
except Exception as ex:
    print(c, sms, "failed", ex)
PY
    done
  done
done
