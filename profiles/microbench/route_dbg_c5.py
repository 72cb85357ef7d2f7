import os; os.environ["PIKV_DEBUG_CTL"] = "1"  # route timestamps (dbg slots 0-5)
import ctypes, sys, numpy as np, torch
sys.path.insert(0,'.')
from bench import make_config, WORKLOADS
from paper_2508_06526_b200.engine import Engine
from paper_2508_06526_b200 import _capi
w=dict(WORKLOADS['c5'][1]); w['L']=2048
cfg=make_config(w)
eng=Engine(cfg)
eng.prefill_synthetic(256, seed=3)
q=torch.empty(64,1024,dtype=torch.bfloat16,device='cuda'); k=torch.empty_like(q); v=torch.empty_like(q)
L=_capi.lib(); L.pikv_debug_read.argtypes=[ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
for i in range(5):
    eng.fill_synthetic(q,k,v,seed=i); eng.step(q,k,v); eng.sync()
    d=np.zeros(64,dtype=np.int64); L.pikv_debug_read(eng.h, d.ctypes.data, 64)
    print("qload %d chain %d (wait %d) sync %d select+writeback %d cycles"%(d[1]-d[0], d[2]-d[1], d[5], d[3]-d[2], d[4]-d[3]))
    print("  select: nan %d penalty %d topk+gates %d note %d cand %d tail %d"%(d[10]-d[3], d[11]-d[10], d[12]-d[11], d[13]-d[12], d[14]-d[13], d[4]-d[14]))
eng.close()
