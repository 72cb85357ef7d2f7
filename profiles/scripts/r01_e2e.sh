set -x
timeout 900 python -m pytest tests/test_group_gpu.py -x -q > gpurun_out/gpu_tests.log 2>&1; echo GT $?
for c in c2 c3 c5; do
  timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline > gpurun_out/e_${c}.log 2>&1
done
timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline --micro 4 > gpurun_out/e_c2_m4.log 2>&1
