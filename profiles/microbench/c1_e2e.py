import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2508_06526_b200.engine import Engine
from paper_2508_06526_b200 import _capi
w = dict(bench.WORKLOADS["c1"][1])
cfg = bench.make_config(w)
eng = Engine(cfg)
eng.prefill_synthetic(w["L"], seed=7)
B, d, dp = cfg.batch, cfg.model.d, cfg.stored_width
hq = torch.randn(3, B, d).pin_memory()
hy = torch.empty(B, dp).pin_memory()
q = hq.cuda()
y = torch.empty(B, dp, device="cuda")
for i in range(5): eng.step(q[0], q[1], q[2], None, y)
eng.sync()
L = _capi.lib()
ts = []
for i in range(30):
    a = time.perf_counter()
    _capi.check(L.pikv_step_host(eng.h, hq[0].data_ptr(), hq[1].data_ptr(), hq[2].data_ptr(), None, hy.data_ptr()))
    ts.append((time.perf_counter() - a) * 1e3)
print(os.environ.get("TAG", ""), "step_host ms", np.round(ts[:6], 3), "median", np.median(ts))
