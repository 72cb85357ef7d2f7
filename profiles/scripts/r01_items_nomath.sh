# k_attend with the consumer math compiled out (PIKV_ATTEND_NOMATH build in
# libpikv_b200_nomath.so): work items per CTA 1 / 4 / 16
cp paper_2508_06526_b200/libpikv_b200_nomath.so paper_2508_06526_b200/libpikv_b200.so
for it in 1 4 16; do
  PIKV_ITEMS=$it python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/nomath_items_$it.log 2>&1
done
