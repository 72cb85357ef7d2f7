#!/bin/bash
# c4-lowrank: repeats of CUDA-core @104 vs HMMA @104 / @116 / @124 attention SMs (run on the GPU box)
set -u
mkdir -p gpurun_out
for r in 1 2 3; do
  for spec in cc:104 tc:104 tc:116 tc:124; do
    k=${spec%%:*}; sms=${spec#*:}
    if [ $k = tc ]; then export PIKV_BF16TC=1; else unset PIKV_BF16TC; fi
    python bench.py --config c4-lowrank --steps 30 --warmup 5 --no-cpu-baseline --attend-sms $sms > gpurun_out/lr_${k}_${sms}_$r.json 2> /dev/null
    python - "gpurun_out/lr_${k}_${sms}_$r.json" "$k" "$sms" <<'PY'
import json, sys
f, k, sms = sys.argv[1:4]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print("%s sms %4s %9.0f tok/s %7.4f ms  attend %.4f ms frac %.3f share %.3f  e2e %9.0f" % (k, sms, d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["roofline"]["attend_share_of_step"], d["e2e"]["value"]))
except Exception as ex:
    print(k, sms, "failed", ex)
PY
  done
done
