set -x
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q -k "lossless or c2_shape or c5_shape or multikernel or embedding" > gpurun_out/gpu_tests.log 2>&1; echo GT $?
timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline > gpurun_out/rp_c2.log 2>&1
timeout 300 python bench.py --config c5 --steps 30 --no-cpu-baseline > gpurun_out/rp_c5.log 2>&1
timeout 300 python bench.py --config c5 --batch 16 --prefill 32768 --retain 0.25 --steps 20 --no-cpu-baseline > gpurun_out/rp_c5_b16.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_route -c 6 --launch-skip 20 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/rp_ncu.log 2>&1
