#!/bin/bash
# Round-2 (second session, final, partition + 4 micro-batches) sweep on one B200 (run by gpurun from the repo root): GPU tests,
# smoke, every workload's bench line, the sharded rehearsal, the reference
# arm, the c2 launch list and one ncu --set full capture of k_attend.
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02e_gpu_all.log 2>&1; echo rc=$? >> gpurun_out/r02e_gpu_all.log
tail -2 gpurun_out/r02e_gpu_all.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02e_smoke.log 2>&1; tail -1 gpurun_out/r02e_smoke.log
for c in c2 c1 c3 c4-int8 c4-int4 c4-lowrank c5; do
  python bench.py --config $c > gpurun_out/r02e_bench_$c.json 2> gpurun_out/r02e_bench_$c.err
  python - $c <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open("gpurun_out/r02e_bench_%s.json" % c).read().strip().splitlines()[-1])
    print("%-11s %9.0f tok/s %7.4f ms attend %.3f e2e %9.0f clocks %s" % (c, d["value"], d["ms_per_step"],
          d["roofline"]["frac"], d["e2e"]["value"], d["clocks"].get("sm_mhz")))
except Exception as ex:
    print(c, "failed", ex)
PY
done
for c in c2 c3; do
  python bench.py --config $c --sharded-rehearsal --no-cpu-baseline > gpurun_out/r02e_bench_${c}_sharded.json 2> gpurun_out/r02e_bench_${c}_sharded.err
  tail -c 160 gpurun_out/r02e_bench_${c}_sharded.json
done
python bench.py --impl reference --steps 10 --warmup 1 > gpurun_out/r02e_ref_c2.json 2> gpurun_out/r02e_ref_c2.err
tail -c 200 gpurun_out/r02e_ref_c2.json
PIKV_GREEN=0 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02e_launch_list.csv python bench.py --steps 3 --warmup 3 --ncu-window --no-cpu-baseline > gpurun_out/r02e_ncu_launch.log 2>&1
echo launch-list rc=$?
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_attend -c 1 \
    -o gpurun_out/r02e_c2_attend python bench.py --steps 3 --warmup 3 --ncu-window --no-cpu-baseline > gpurun_out/r02e_ncu_full.log 2>&1
echo ncu-full rc=$?
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_attend_bf16tc -c 1 \
    -o gpurun_out/r02e_lowrank_attend python bench.py --config c4-lowrank --steps 3 --warmup 3 --ncu-window --no-cpu-baseline > gpurun_out/r02e_ncu_full_lr.log 2>&1
echo ncu-full-lowrank rc=$?
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_attend_i4tc -c 1 \
    -o gpurun_out/r02e_int4_attend python bench.py --config c4-int4 --steps 3 --warmup 3 --ncu-window --no-cpu-baseline > gpurun_out/r02e_ncu_full_i4.log 2>&1
echo ncu-full-int4 rc=$?
