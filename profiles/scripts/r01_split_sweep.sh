# k_attend: bulk copies per KV entry (PIKV_SPLIT)
for sp in 1 2 4 8; do
  PIKV_SPLIT=$sp python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/split_$sp.log 2>&1
done
