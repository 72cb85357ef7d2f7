set -x
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_group_gpu.py tests/test_multirank_gpu.py -x -q > gpurun_out/gpu_tests.log 2>&1; echo GT $?
PIKV_CONTROL=0 python profiles/microbench/route_dbg.py > gpurun_out/rdbg.log 2>&1
PIKV_CONTROL=0 python profiles/microbench/route_dbg_c5.py > gpurun_out/rdbg5.log 2>&1
timeout 300 python bench.py --config c5 --batch 16 --prefill 32768 --retain 0.25 --steps 20 --no-cpu-baseline > gpurun_out/rp5.log 2>&1
timeout 300 python bench.py --config c1 --steps 30 --no-cpu-baseline > gpurun_out/rp1.log 2>&1
