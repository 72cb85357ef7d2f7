set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_route|k_sched_select|k_retr_scan|k_foldback|k_combine|k_retr_write|k_insert" -c 7 --launch-skip 70 \
  -o gpurun_out/ctl_c2 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_ctl.log 2>&1; echo NCU $?
