# SPDX-License-Identifier: Apache-2.0
"""A/B inside one process: the micro-batch e2e host loop with and without the
attention timing events (pikv_group_set_timing), alternating runs.
python profiles/microbench/e2e_timing_ab.py [config]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_06526_b200 import _capi  # noqa: E402
from paper_2508_06526_b200.engine import EngineGroup  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = dict(bench.WORKLOADS[name][1])
cfg = bench.make_config(w)
grp = EngineGroup(cfg, n_micro=2, attend_sms=0)
grp.prefill_synthetic(w["L"], seed=7)
B, d, dp, Bm, n = cfg.batch, cfg.model.d, cfg.stored_width, grp.Bm, 2
steps = 50
hq = torch.randn(steps, n, 3, Bm, d).to(torch.bfloat16).pin_memory()
hy = torch.empty(B, dp, dtype=torch.float32).pin_memory()
L = _capi.lib()
h = grp.h
yptr = [hy[m * Bm].data_ptr() for m in range(n)]
st0 = grp.engines[0].external_stream()


def run():
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st0)
    for i in range(steps):
        for m in range(n):
            if i:
                _capi.check(L.pikv_group_wait(h, m))
            _capi.check(L.pikv_group_submit(h, m, hq[i, m, 0].data_ptr(), hq[i, m, 1].data_ptr(),
                                            hq[i, m, 2].data_ptr(), None, yptr[m], 1))
    for m in range(n):
        _capi.check(L.pikv_group_wait(h, m))
    grp.join()
    e1.record(st0)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


res = {"off": [], "on": []}
run()
for rep in range(4):
    for mode in ("off", "on"):
        grp.set_timing(mode == "on")
        res[mode].append(run())
        grp.set_timing(False)
        grp.read_timing()
print({k: [round(x, 4) for x in v] for k, v in res.items()},
      {k: round(float(np.median(v)), 4) for k, v in res.items()})
grp.close()
