set -x
timeout 900 python -m pytest tests/test_ops_gpu.py tests/test_engine_gpu.py -x -q > gpurun_out/gpu_tests.log 2>&1; echo GT $?
for c in c4-int8 c4-int4; do
  timeout 300 python bench.py --config $c --steps 30 --no-cpu-baseline --micro 1 > gpurun_out/t_${c}_m1.log 2>&1
done
for c in c2 c5 c4-lowrank; do
  timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline > gpurun_out/t_${c}.log 2>&1
done
timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline --micro 1 > gpurun_out/t_c2_m1.log 2>&1
