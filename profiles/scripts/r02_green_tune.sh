#!/bin/bash
# attention SM partition: partition size and shares vs tickets (run on the GPU box)
set -u
mkdir -p gpurun_out
run() {  # label config env...
  local lab=$1 c=$2; shift 2
  env "$@" python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline ${EXTRA:-} > gpurun_out/gt2.json 2>/dev/null
  python - "$lab" "$c" <<'PY'
import json, sys
lab, c = sys.argv[1:3]
try:
    d = json.loads(open("gpurun_out/gt2.json").read().strip().splitlines()[-1])
    r = d["roofline"]
    print("%-14s %-8s %9.0f tok/s %7.4f ms  frac %.3f busy %.4f  e2e %9.0f" % (lab, c, d["value"], d["ms_per_step"], r["frac"], r["busy_ms_per_launch"], d["e2e"]["value"]))
except Exception as ex:
    print(lab, c, "failed", ex)
PY
}
for r in 1 2; do
  for sms in 96 104 112 120; do EXTRA="--attend-sms $sms" run "sms$sms" c2 PIKV_GREEN=1; done
  for c in c2 c3 c5 c4-int8; do
    run share $c PIKV_ATT_SHARE=1
    run tickets $c PIKV_ATT_SHARE=0
  done
done
