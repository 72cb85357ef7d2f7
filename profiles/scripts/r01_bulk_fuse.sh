set -x
timeout 900 python -m pytest tests/test_bulk_gpu.py tests/test_replay_gpu.py -x -q > gpurun_out/bulk_tests.log 2>&1; echo BT $?
PIKV_BULK_FUSE=0 timeout 900 python -m pytest tests/test_bulk_gpu.py -x -q > gpurun_out/bulk_tests_nf.log 2>&1; echo BT0 $?
timeout 300 python profiles/microbench/bulk_bench.py 32768 > gpurun_out/bulk_fuse.log 2>&1
PIKV_BULK_FUSE=0 timeout 300 python profiles/microbench/bulk_bench.py 32768 > gpurun_out/bulk_nofuse.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_bulk|k_basis" -c 8 --log-file gpurun_out/bulk_ll7.csv python profiles/microbench/bulk_bench.py 32768 > gpurun_out/bulk_ll7.log 2>&1
