#!/bin/bash
# A/B of k_attend build variants (attend.cu macros) on the bench configs.
# usage: profiles/scripts/ab_attend.sh "<label>:<nvcc flags>" ...   (run on the GPU box)
set -u
mkdir -p gpurun_out
for spec in "$@"; do
  label=${spec%%:*}; flags=${spec#*:}
  PIKV_NVCC_FLAGS="$flags" python -m paper_2508_06526_b200.build -f > /dev/null || { echo "$label build failed"; continue; }
  for c in c2 c4-int8 c4-int4 c4-lowrank; do
    python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${label}_$c.json 2> gpurun_out/ab_${label}_$c.err
    python - "$label" "$c" <<'PY'
import json, sys
label, c = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open("gpurun_out/ab_%s_%s.json" % (label, c)).read().strip().splitlines()[-1])
    print("%-10s %-11s %8.0f tok/s %7.4f ms  attend frac %.3f  e2e %8.0f" % (label, c, d["value"], d["ms_per_step"], d["roofline"]["frac"], d["e2e"]["value"]))
except Exception as ex:
    print(label, c, "failed", ex)
PY
  done
done
