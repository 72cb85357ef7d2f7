set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo GT $?
for c in c4-int8 c4-int4; do
  timeout 300 python bench.py --config $c --steps 30 --no-cpu-baseline --micro 1 > gpurun_out/s_${c}_m1.log 2>&1
  timeout 300 python bench.py --config $c --steps 30 --no-cpu-baseline --micro 2 --attend-sms 148 > gpurun_out/s_${c}_m2.log 2>&1
done
for c in c2 c5 c4-lowrank; do
  timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline > gpurun_out/s_${c}.log 2>&1
done
timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline --micro 1 > gpurun_out/s_c2_m1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attend -c 1 --launch-skip 3 \
  -o gpurun_out/att3_c4-int4 -f python bench.py --config c4-int4 --micro 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1; echo NCU $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attend -c 1 --launch-skip 3 \
  -o gpurun_out/att3_c4-int8 -f python bench.py --config c4-int8 --micro 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3b.log 2>&1; echo NCU $?
