#!/bin/bash
# c4-lowrank on the bf16 tensor-core kernel: stage size (8 / 16 entries) and
# attention-SM A/B against the CUDA-core kernel; one ncu --set full capture
mkdir -p gpurun_out
summ() { python - "$1" "$2" <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
print(sys.argv[2], round(d["value"]), round(d["ms_per_step"], 4), "attend", round(d["roofline"]["avg_launch_ms"], 4), round(d["roofline"]["frac"], 3), "e2e", round(d["e2e"]["value"]))
PY
}
for s in 104 124; do
  timeout 300 python bench.py --config c4-lowrank --attend-sms $s --steps 30 --no-cpu-baseline > gpurun_out/btc8_$s.json 2>/dev/null; summ gpurun_out/btc8_$s.json "tc eps8 sms $s"
  PIKV_BF16TC_EPS=16 timeout 300 python bench.py --config c4-lowrank --attend-sms $s --steps 30 --no-cpu-baseline > gpurun_out/btc16_$s.json 2>/dev/null; summ gpurun_out/btc16_$s.json "tc eps16 sms $s"
  PIKV_BF16TC=0 timeout 300 python bench.py --config c4-lowrank --attend-sms $s --steps 30 --no-cpu-baseline > gpurun_out/bcc_$s.json 2>/dev/null; summ gpurun_out/bcc_$s.json "cc sms $s"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attend_bf16tc -c 1 --launch-skip 3 \
  -o gpurun_out/btc_c4lr -f python bench.py --config c4-lowrank --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/btc_ncu.log 2>&1; echo NCU $?
