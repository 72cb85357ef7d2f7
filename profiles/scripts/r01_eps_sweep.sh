# k_attend entries-per-stage sweep (PIKV_EPS; stages = 110 KB / stage bytes)
for eps in 1 2 3; do
  PIKV_EPS=$eps python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/eps_$eps.log 2>&1
  PIKV_EPS=$eps python bench.py --config c5 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/eps_c5_$eps.log 2>&1
done
