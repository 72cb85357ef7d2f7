set -x
timeout 900 python -m pytest tests/test_engine_gpu.py -x -q -k "codecs or quant or c2_shape" > gpurun_out/gpu_tests.log 2>&1; echo GT $?
timeout 300 python bench.py --config c4-int8 --steps 30 --no-cpu-baseline > gpurun_out/i_c4-int8.log 2>&1
timeout 300 python bench.py --config c4-int8 --steps 30 --no-cpu-baseline --micro 1 > gpurun_out/i_c4-int8_m1.log 2>&1
timeout 300 python bench.py --config c1 --steps 30 --no-cpu-baseline > gpurun_out/i_c1.log 2>&1
PIKV_PDL=1 timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline > gpurun_out/i_c2_pdl.log 2>&1
timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline > gpurun_out/i_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attend -c 1 --launch-skip 3 \
  -o gpurun_out/att4_c4-int8 -f python bench.py --config c4-int8 --micro 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu4.log 2>&1; echo NCU $?
