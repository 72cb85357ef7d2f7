# Round-1 measurement sweep (run on the GPU box from the repo root; outputs to gpurun_out/)
set -x
python bench.py > gpurun_out/r01_bench_default.log 2>&1
python bench.py --impl reference > gpurun_out/r01_bench_ref.log 2>&1
for c in c1 c3 c4-int8 c4-int4 c4-lowrank c5; do
  python bench.py --config $c --steps 30 --no-cpu-baseline > gpurun_out/r01_bench_$c.log 2>&1
done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --ncu-window > gpurun_out/r01_ncu_dry.log 2>&1; echo DRY $?
