set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo GT $?
for c in c4-int8 c4-int4; do
  for m in 1 2; do
  timeout 300 python bench.py --config $c --steps 30 --no-cpu-baseline --micro $m > gpurun_out/q_${c}_m$m.log 2>&1
  done
done
for c in c2 c5 c4-lowrank c3; do
  timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline > gpurun_out/q_${c}.log 2>&1
done
timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline --micro 1 > gpurun_out/q_c2_m1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attend -c 1 --launch-skip 3 \
  -o gpurun_out/att2_c4-int8 -f python bench.py --config c4-int8 --micro 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo NCU $?
