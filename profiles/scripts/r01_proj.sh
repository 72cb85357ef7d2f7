set -x
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_group_gpu.py -x -q -k "codecs or group or LowRank" > gpurun_out/gpu_tests.log 2>&1; echo GT $?
timeout 300 python bench.py --config c4-lowrank --steps 30 --no-cpu-baseline > gpurun_out/k_c4-lowrank.log 2>&1
timeout 300 python bench.py --config c4-lowrank --steps 30 --no-cpu-baseline --attend-sms 124 > gpurun_out/k_c4-lowrank_a124.log 2>&1
timeout 300 python bench.py --config c4-lowrank --steps 30 --no-cpu-baseline --attend-sms 96 > gpurun_out/k_c4-lowrank_a96.log 2>&1
