set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo GT $?
for c in c2 c3 c5 c4-lowrank; do
  for p in 0 1; do
    PIKV_ATT_STATIC=$p timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline > gpurun_out/dy_${c}_s$p.log 2>&1
  done
done
PIKV_ATT_STATIC=0 timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline --micro 1 > gpurun_out/dy_c2_m1.log 2>&1
for a in 132 140 148; do
timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline --attend-sms $a > gpurun_out/dy_c2_a$a.log 2>&1
done
