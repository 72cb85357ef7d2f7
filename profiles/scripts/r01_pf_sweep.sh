# L2 prefetch distance sweep for k_attend (PIKV_PF entries ahead)
for pf in 0 2 4 8 16; do
  PIKV_PF=$pf python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/pf_$pf.log 2>&1
done
