set -x
for a in 100 108 112 120; do
  timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline --attend-sms $a > gpurun_out/se_c2_a$a.log 2>&1
done
for a in 104 120 132; do
  timeout 300 python bench.py --config c4-lowrank --steps 30 --no-cpu-baseline --attend-sms $a > gpurun_out/se_lr_a$a.log 2>&1
done
for a in 104 120; do
  timeout 300 python bench.py --config c5 --steps 30 --no-cpu-baseline --attend-sms $a > gpurun_out/se_c5_a$a.log 2>&1
done
