#!/bin/bash
# c4-int8 with static shares: attention SMs sweep (run on the GPU box)
set -u
mkdir -p gpurun_out
for r in 1 2; do
  for sms in 124 130 136 142 148; do
    python bench.py --config c4-int8 --steps 100 --warmup 5 --no-cpu-baseline --attend-sms $sms > gpurun_out/i8_${sms}_$r.json 2> /dev/null
    python - "gpurun_out/i8_${sms}_$r.json" "$sms" <<'PY'
import json, sys
f, sms = sys.argv[1:3]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print("c4-int8 sms %4s %9.0f tok/s %7.4f ms  attend %.4f ms frac %.3f share %.3f  e2e %9.0f" % (sms, d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["roofline"]["attend_share_of_step"], d["e2e"]["value"]))
except Exception as ex:
    print(sms, "failed", ex)
PY
  done
done
