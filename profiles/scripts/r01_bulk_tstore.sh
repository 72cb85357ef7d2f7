set -x
timeout 600 python -m pytest tests/test_bulk_gpu.py -x -q > gpurun_out/bulk_tests.log 2>&1; echo BT $?
timeout 300 python profiles/microbench/bulk_bench.py 32768 > gpurun_out/bulk_ts.log 2>&1
PIKV_BULK_TSTORE=0 timeout 300 python profiles/microbench/bulk_bench.py 32768 > gpurun_out/bulk_ts0.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bulk_project_tc3 -c 1 --launch-skip 1 -o gpurun_out/bulk_tc3s -f python profiles/microbench/bulk_bench.py 32768 > gpurun_out/bulk_ncu3s.log 2>&1; echo NCU $?
