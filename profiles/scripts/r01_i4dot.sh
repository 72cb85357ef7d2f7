set -x
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_ops_gpu.py tests/test_bulk_gpu.py -x -q -k "codecs or quant or Int or int" > gpurun_out/gpu_tests.log 2>&1; echo GT $?
timeout 300 python bench.py --config c4-int4 --steps 30 --no-cpu-baseline > gpurun_out/j_c4-int4.log 2>&1
timeout 300 python bench.py --config c4-int4 --steps 30 --no-cpu-baseline --micro 1 > gpurun_out/j_c4-int4_m1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attend -c 1 --launch-skip 3 \
  -o gpurun_out/att5_c4-int4 -f python bench.py --config c4-int4 --micro 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu5.log 2>&1; echo NCU $?
