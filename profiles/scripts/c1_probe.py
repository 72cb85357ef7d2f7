"""c1 step anatomy: k_control phase stamps (PIKV_DEBUG_CTL=1, globaltimer ns)
and the eager per-kernel phase times of the single-engine c1 step."""
import ctypes
import os
import sys

os.environ["PIKV_DEBUG_CTL"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_06526_b200 import _capi  # noqa: E402
from paper_2508_06526_b200.engine import Engine  # noqa: E402

w = bench.WORKLOADS["c1"][1]
cfg = bench.make_config(w)
eng = Engine(cfg)
eng.prefill_synthetic(w["L"], seed=7)
B, d = cfg.batch, cfg.model.d
qkv = torch.empty(3, B, d, dtype=torch.float32, device="cuda")
y = torch.empty(B, cfg.stored_width, dtype=torch.float32, device="cuda")
L = _capi.lib()
L.pikv_debug_read.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong), ctypes.c_int]
buf = (ctypes.c_longlong * (64 + 8 * B))()
names = ["route", "insert+sync", "sched", "retrieve", "items"]
acc = np.zeros(5)
n = 0
for i in range(40):
    eng.fill_synthetic(qkv[0], qkv[1], qkv[2], seed=1000 + i)
    eng.step(qkv[0], qkv[1], qkv[2], None, y)
    eng.sync()
    L.pikv_debug_read(eng.h, buf, 64 + 8 * B)
    st = [buf[64 + p] for p in range(6)]
    if i >= 10 and all(st):
        acc += np.diff(np.array(st, dtype=np.float64)) / 1e3
        n += 1
print("k_control phases (us, stream 0, mean of %d):" % n, {k: round(v / max(n, 1), 2) for k, v in zip(names, acc)})
eng.set_profiling(True)
for i in range(20):
    eng.step(qkv[0], qkv[1], qkv[2], None, y)
phases, nl = eng.read_profile()
eng.set_profiling(False)
print("eager phases (us):", {k: round(1e3 * v / max(nl, 1), 1) for k, v in phases.items()})
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
es = eng.external_stream()
torch.cuda.synchronize()
ev0.record(es)
for i in range(200):
    eng.step(qkv[0], qkv[1], qkv[2], None, y)
ev1.record(es)
torch.cuda.synchronize()
print("graph step: %.1f us" % (ev0.elapsed_time(ev1) * 1e3 / 200))
