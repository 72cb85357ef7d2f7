set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo GT $?
for c in c4-lowrank c2 c5; do
  timeout 300 python bench.py --config $c --steps 30 --no-cpu-baseline > gpurun_out/nb_$c.log 2>&1
done
timeout 300 python bench.py --config c4-lowrank --steps 30 --no-cpu-baseline --micro 1 > gpurun_out/nb_c4-lowrank_m1.log 2>&1
