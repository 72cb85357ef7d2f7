#!/bin/bash
# k_attend: one bulk copy per run of pool-adjacent entries (PIKV_ATT_MERGE=1)
# vs one per entry
mkdir -p gpurun_out
summ() { python - "$1" "$2" <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
print(sys.argv[2], round(d["value"]), round(d["ms_per_step"], 4), "attend", round(d["roofline"]["avg_launch_ms"], 4), round(d["roofline"]["frac"], 3), "e2e", round(d["e2e"]["value"]))
PY
}
for c in c2 c4-lowrank c4-int8; do
  for m in 0 1; do
    PIKV_ATT_MERGE=$m timeout 300 python bench.py --config $c --steps 30 --no-cpu-baseline > gpurun_out/mg_${c}_$m.json 2>/dev/null; summ gpurun_out/mg_${c}_$m.json "$c merge=$m"
  done
done
