set -x
timeout 600 python -m pytest tests/test_group_gpu.py -x -q > gpurun_out/group_tests.log 2>&1; echo GT $?
for c in c2 c3 c5; do
  for p in 0 1; do
    PIKV_ATT_PRIO=$p timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline > gpurun_out/pr_${c}_p$p.log 2>&1
  done
done
for a in 132 140; do
timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline --attend-sms $a > gpurun_out/pr_c2_a$a.log 2>&1
done
