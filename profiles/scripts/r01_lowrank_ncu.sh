# c4-lowrank attention: launch list + one ncu --set full of k_attend (run from the repo root on the GPU box)
set -x
timeout 300 python bench.py --config c4-lowrank --steps 30 --no-cpu-baseline > gpurun_out/lr_bench.log 2>&1; echo B $?
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/lr_launch_list.csv python bench.py --config c4-lowrank --steps 2 --warmup 3 --no-cpu-baseline --ncu-window > gpurun_out/lr_ncu_ll.log 2>&1; echo LL $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attend -c 1 --launch-skip 6 \
  -o gpurun_out/lr_attend -f python bench.py --config c4-lowrank --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/lr_ncu_full.log 2>&1; echo NF $?
