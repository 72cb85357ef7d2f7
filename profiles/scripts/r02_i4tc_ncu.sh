#!/bin/bash
# ncu --set full of the tensor-core int4 attention kernel (c4-int4, one
# micro-batch launch after warm-up), source-mapped
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attend_i4tc -c 1 --launch-skip 3 \
  -o gpurun_out/i4tc_c4 -f python bench.py --config c4-int4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/i4tc_ncu.log 2>&1; echo NCU $?
