set -x
for f in 0 1; do
  PIKV_RETR_FUSED=$f timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline > gpurun_out/f_c2_rf$f.log 2>&1
done
for a in 116 108; do
  timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline --attend-sms $a > gpurun_out/f_c2_a$a.log 2>&1
done
PIKV_RETR_FUSED=1 timeout 300 python bench.py --config c5 --steps 50 --no-cpu-baseline > gpurun_out/f_c5_rf1.log 2>&1
timeout 300 python bench.py --config c5 --steps 50 --no-cpu-baseline > gpurun_out/f_c5_rf0.log 2>&1
