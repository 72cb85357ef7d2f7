set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo GT $?
timeout 400 python bench.py --config c2 --batch 1 --steps 30 --no-cpu-baseline > gpurun_out/cb_c2_b1.log 2>&1
timeout 400 python bench.py --config c2 --steps 50 --no-cpu-baseline > gpurun_out/cb_c2.log 2>&1
timeout 400 python bench.py --config c5 --batch 16 --prefill 32768 --retain 0.25 --steps 20 --no-cpu-baseline > gpurun_out/cb_c5_b16.log 2>&1
