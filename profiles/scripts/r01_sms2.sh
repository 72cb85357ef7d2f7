set -x
for a in 112 124 136 148; do
  timeout 300 python bench.py --config c4-int8 --steps 30 --no-cpu-baseline --attend-sms $a > gpurun_out/s2_i8_a$a.log 2>&1
done
for a in 136 148; do
  timeout 300 python bench.py --config c4-int4 --steps 30 --no-cpu-baseline --attend-sms $a > gpurun_out/s2_i4_a$a.log 2>&1
done
for a in 100 124; do
  timeout 300 python bench.py --config c3 --steps 50 --no-cpu-baseline --attend-sms $a > gpurun_out/s2_c3_a$a.log 2>&1
done
