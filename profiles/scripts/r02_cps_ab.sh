#!/bin/bash
# A/B: two vs three attention CTAs per SM (PIKV_ATT_CPS) x attention SMs (run on the GPU box)
set -u
mkdir -p gpurun_out
for c in ${1:-c4-lowrank c2}; do
  for cps in 2 3; do
    for sms in ${2:-104}; do
      PIKV_ATT_CPS=$cps python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --attend-sms $sms > gpurun_out/cps_${cps}_${sms}_$c.json 2> gpurun_out/cps_${cps}_${sms}_$c.err
      python - "$cps" "$sms" "$c" <<'PY'
import json, sys
cps, sms, c = sys.argv[1:4]
try:
    d = json.loads(open("gpurun_out/cps_%s_%s_%s.json" % (cps, sms, c)).read().strip().splitlines()[-1])
    print("cps %s sms %4s %-11s %9.0f tok/s %7.4f ms  attend %.4f ms frac %.3f share %.3f  e2e %9.0f" % (cps, sms, c, d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["roofline"]["attend_share_of_step"], d["e2e"]["value"]))
except Exception as ex:
    print(cps, sms, c, "failed", ex)
PY
    done
  done
done
