#!/bin/bash
# attention-grid SM count sweep (the rest of the SMs run the other
# micro-batch's control kernels) for c4-int4 after the tensor-core kernel
mkdir -p gpurun_out
for s in 136 128 120 112 100; do
  timeout 300 python bench.py --config c4-int4 --attend-sms $s --steps 30 --no-cpu-baseline > gpurun_out/sms_i4_$s.json 2>/dev/null
  python - "$s" <<'PY'
import json, sys
d = json.loads([l for l in open("gpurun_out/sms_i4_%s.json" % sys.argv[1]) if l.startswith("{")][-1])
print("c4-int4 sms", sys.argv[1], round(d["value"]), round(d["ms_per_step"], 4), "attend", round(d["roofline"]["avg_launch_ms"], 4), "e2e", round(d["e2e"]["value"]))
PY
done
