set -x
for c in c4-int8 c4-int4; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attend -c 1 --launch-skip 3 \
  -o gpurun_out/att_$c -f python bench.py --config $c --micro 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$c.log 2>&1; echo $c $?
done
for it in 1 2 8; do
PIKV_ITEMS=$it timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline > gpurun_out/it_c2_$it.log 2>&1
done
