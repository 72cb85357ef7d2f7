# clock64 checkpoints inside k_sched_select for (stream 0, 1) on c2 after prefill
import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
from bench import make_config, WORKLOADS
from paper_2508_06526_b200.engine import Engine
from paper_2508_06526_b200 import _capi
w = dict(WORKLOADS['c2'][1])
cfg = make_config(w)
eng = Engine(cfg)
eng.prefill_synthetic(w['L'], seed=3)
q = torch.empty(16, 4096, dtype=torch.bfloat16, device='cuda'); k = torch.empty_like(q); v = torch.empty_like(q)
L = _capi.lib(); L.pikv_debug_read.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
for i in range(12):
    eng.fill_synthetic(q, k, v, seed=i); eng.step(q, k, v); eng.sync()
    d = np.zeros(64, dtype=np.int64); L.pikv_debug_read(eng.h, d.ctypes.data, 64)
    for sg in (0, 1):
        t = d[16 + 8 * sg: 24 + 8 * sg]
        print("sg%d V=%d stage %d count %d argmin %d erase %d (cycles)" % (sg, t[6], t[1] - t[0], t[2] - t[1], t[3] - t[2], t[4] - t[3]))
eng.close()
