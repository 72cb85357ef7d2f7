# c4-lowrank attention A/B: chunks per thread (PIKV_ATT_CPT) and attention grid SMs
set -x
for r in 1 2; do
timeout 300 python bench.py --config c4-lowrank --steps 30 --no-cpu-baseline > gpurun_out/ab_lr_base_$r.log 2>&1
for c in 2 4; do
  PIKV_ATT_CPT=$c timeout 300 python bench.py --config c4-lowrank --steps 30 --no-cpu-baseline > gpurun_out/ab_lr_cpt${c}_$r.log 2>&1
done
for a in 80 88 96; do
  timeout 300 python bench.py --config c4-lowrank --steps 30 --no-cpu-baseline --attend-sms $a > gpurun_out/ab_lr_a${a}_$r.log 2>&1
done
done
