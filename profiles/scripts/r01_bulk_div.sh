set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo GT $?
timeout 300 python profiles/microbench/bulk_bench.py 32768 > gpurun_out/bulk_div.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_bulk|k_basis" -c 5 --log-file gpurun_out/bulk_ll3.csv python profiles/microbench/bulk_bench.py 32768 > gpurun_out/bulk_ll3.log 2>&1
timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline > gpurun_out/div_c2.log 2>&1
timeout 300 python bench.py --config c1 --steps 50 --no-cpu-baseline > gpurun_out/div_c1.log 2>&1
