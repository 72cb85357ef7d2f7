# SPDX-License-Identifier: Apache-2.0
"""Host-side timing of the micro-batch e2e loop (pikv_group_submit(host=1) /
pikv_group_wait): how long each submit call and each wait takes on the host,
next to the device step time.  python profiles/microbench/e2e_diag.py [config]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_06526_b200 import _capi  # noqa: E402
from paper_2508_06526_b200.engine import EngineGroup  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
n_micro = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = dict(bench.WORKLOADS[name][1])
cfg = bench.make_config(w)
grp = EngineGroup(cfg, n_micro=n_micro, attend_sms=0)
grp.prefill_synthetic(w["L"], seed=7)
B, d, dp, Bm = cfg.batch, cfg.model.d, cfg.stored_width, grp.Bm
steps = 60
hq = torch.randn(steps, n_micro, 3, Bm, d).to(torch.bfloat16).pin_memory()
hy = torch.empty(B, dp, dtype=torch.float32).pin_memory()
L = _capi.lib()
h = grp.h
yptr = [hy[m * Bm].data_ptr() for m in range(n_micro)]
t_sub, t_wait = [], []
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(steps):
    for m in range(n_micro):
        if i:
            a = time.perf_counter()
            _capi.check(L.pikv_group_wait(h, m))
            t_wait.append(time.perf_counter() - a)
        a = time.perf_counter()
        _capi.check(L.pikv_group_submit(h, m, hq[i, m, 0].data_ptr(), hq[i, m, 1].data_ptr(),
                                        hq[i, m, 2].data_ptr(), None, yptr[m], 1))
        t_sub.append(time.perf_counter() - a)
grp.sync()
tot = time.perf_counter() - t0
sub = np.array(t_sub[2 * n_micro:]) * 1e6
wt = np.array(t_wait[2 * n_micro:]) * 1e6
print({"config": name, "n_micro": n_micro, "ms_per_step_wall": tot / steps * 1e3,
       "submit_us_median": float(np.median(sub)), "submit_us_p90": float(np.percentile(sub, 90)),
       "wait_us_median": float(np.median(wt)), "wait_us_p90": float(np.percentile(wt, 90))})
grp.close()
