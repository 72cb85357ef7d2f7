# A/B of the per-stream control kernel (default) vs the multi-kernel path (PIKV_CONTROL=0)
for c in c3 c4-int8 c4-lowrank c5 c1; do
  PIKV_DEBUG_CTL=1 python bench.py --config $c --steps 30 --no-cpu-baseline > gpurun_out/ab_ctl_$c.log 2>&1
  PIKV_CONTROL=0 python bench.py --config $c --steps 30 --no-cpu-baseline > gpurun_out/ab_mk_$c.log 2>&1
done
