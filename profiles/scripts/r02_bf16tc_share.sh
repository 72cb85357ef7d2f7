#!/bin/bash
# c4-lowrank: CUDA-core kernel vs the HMMA kernel (PIKV_BF16TC=1) with equal static shares, x attention SMs
set -u
mkdir -p gpurun_out
for k in cc tc; do
  for sms in ${1:-104 116 124 132}; do
    if [ $k = tc ]; then export PIKV_BF16TC=1; else unset PIKV_BF16TC; fi
    python bench.py --config c4-lowrank --steps 30 --warmup 5 --no-cpu-baseline --attend-sms $sms > gpurun_out/btc_${k}_$sms.json 2> gpurun_out/btc_${k}_$sms.err
    python - "$k" "$sms" <<'PY'
import json, sys
k, sms = sys.argv[1:3]
try:
    d = json.loads(open("gpurun_out/btc_%s_%s.json" % (k, sms)).read().strip().splitlines()[-1])
    print("%s sms %4s %9.0f tok/s %7.4f ms  attend %.4f ms frac %.3f share %.3f  e2e %9.0f" % (k, sms, d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["roofline"]["attend_share_of_step"], d["e2e"]["value"]))
except Exception as ex:
    print(k, sms, "failed", ex)
PY
  done
done
