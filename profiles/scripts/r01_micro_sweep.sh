set -x
for a in 148 136 124 112; do
  timeout 300 python bench.py --no-cpu-baseline --steps 50 --attend-sms $a > gpurun_out/sw_c2_a$a.log 2>&1
done
PIKV_CONTROL=1 timeout 300 python bench.py --no-cpu-baseline --steps 50 --attend-sms 124 > gpurun_out/sw_c2_ctl1.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 50 --micro 4 --attend-sms 124 > gpurun_out/sw_c2_m4.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 50 --micro 2 --attend-sms 124 --config c5 > gpurun_out/sw_c5_m2.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 50 --micro 1 --config c5 > gpurun_out/sw_c5_m1.log 2>&1
