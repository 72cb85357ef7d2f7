#!/bin/bash
# A/B of the attention work distribution (run on the GPU box):
#   tickets  = PIKV_ATT_SHARE=0 (round-2 ticketed items)
#   share    = equal static shares, no pool (PIKV_ATT_POOL=0)
#   pool<P>  = static shares + a P % ticketed pool (default 10)
# usage: profiles/scripts/r02_share_ab.sh "c2 c4-lowrank ..." "tickets share pool10 ..."
set -u
mkdir -p gpurun_out
cfgs=${1:-c2 c4-int8 c4-lowrank c3 c5}
vars=${2:-tickets share pool10}
for c in $cfgs; do
  for v in $vars; do
    case $v in
      tickets) env="PIKV_ATT_SHARE=0";;
      share) env="PIKV_ATT_POOL=0";;
      pool*) env="PIKV_ATT_POOL=${v#pool}";;
    esac
    env $env python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/sab_${v}_$c.json 2> gpurun_out/sab_${v}_$c.err
    python - "$v" "$c" <<'PY'
import json, sys
v, c = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open("gpurun_out/sab_%s_%s.json" % (v, c)).read().strip().splitlines()[-1])
    print("%-8s %-11s %9.0f tok/s %7.4f ms  attend %.4f ms frac %.3f share %.3f  e2e %9.0f" % (v, c, d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["roofline"]["attend_share_of_step"], d["e2e"]["value"]))
except Exception as ex:
    print(v, c, "failed", ex)
PY
  done
done
