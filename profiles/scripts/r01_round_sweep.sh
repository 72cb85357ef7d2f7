# Round-1 measurement sweep after the micro-batch pipeline (run from the repo root on the GPU box)
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo GT $?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo SMOKE $?
timeout 400 python bench.py > gpurun_out/r_c2.log 2>&1; echo B $?
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r_ref.log 2>&1; echo R $?
for c in c1 c3 c4-int8 c4-int4 c4-lowrank c5; do
  timeout 300 python bench.py --config $c --steps 30 --no-cpu-baseline > gpurun_out/r_$c.log 2>&1
done
timeout 300 python bench.py --micro 1 --no-cpu-baseline > gpurun_out/r_c2_m1.log 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r_launch_list.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --ncu-window > gpurun_out/r_ncu_ll.log 2>&1; echo LL $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attend -c 1 --launch-skip 6 \
  -o gpurun_out/r_attend_c2 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r_ncu_full.log 2>&1; echo NF $?
