set -x
timeout 600 python -m pytest tests/test_group_gpu.py -x -q > gpurun_out/group_tests.log 2>&1; echo GT $?
timeout 400 python bench.py > gpurun_out/g_c2.log 2>&1; echo B $?
for c in c3 c4-int8 c4-int4 c4-lowrank c5; do
  timeout 300 python bench.py --config $c --steps 30 --no-cpu-baseline > gpurun_out/g_$c.log 2>&1
done
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/g_launch_list.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --ncu-window > gpurun_out/g_ncu.log 2>&1; echo NCU $?
