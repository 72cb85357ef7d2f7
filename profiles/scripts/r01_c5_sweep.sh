# BASELINE configs[4] sweep at 1 GPU: E64 top-4, 8 heads x 128 bf16, batch x context,
# retaining 25% of entries from 32K (SURVEY 8 d, config 5); infeasible points skipped
# (B256 x L128K retained = 137 GB of KV).  One bench line per point.
set -x
for pt in "4096 1 1.0" "4096 16 1.0" "4096 64 1.0" "4096 256 1.0" \
          "32768 1 0.25" "32768 16 0.25" "32768 64 0.25" "32768 256 0.25" \
          "131072 1 0.25" "131072 16 0.25" "131072 64 0.25"; do
  set -- $pt
  timeout 500 python bench.py --config c5 --prefill $1 --batch $2 --retain $3 --steps 20 --warmup 3 \
    --no-cpu-baseline > gpurun_out/sw5_L$1_B$2.log 2>&1; echo "L=$1 B=$2 rc=$?"
done
timeout 300 python bench.py --config c3 --steps 30 --no-cpu-baseline > gpurun_out/sw5_c3.log 2>&1
