"""Per-stream phase timestamps of k_control (PIKV_DEBUG_CTL=1): c2 engine
prefilled to L, then a few decode steps; prints per phase the max over
streams and the kernel span."""
import ctypes, os, sys
import numpy as np, torch
os.environ["PIKV_DEBUG_CTL"] = "1"
sys.path.insert(0, '.')
from bench import make_config, WORKLOADS
from paper_2508_06526_b200.engine import Engine
from paper_2508_06526_b200 import _capi
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = dict(WORKLOADS[name][1])
cfg = make_config(w)
B, d = w["B"], w["H"] * w["hd"]
eng = Engine(cfg)
eng.prefill_synthetic(w["L"], seed=3)
dt = torch.bfloat16 if cfg.kv_dtype == "bf16" else torch.float32
q = torch.empty(B, d, dtype=dt, device='cuda'); k = torch.empty_like(q); v = torch.empty_like(q)
L = _capi.lib(); L.pikv_debug_read.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
names = ["route", "insert", "sched", "retrieve", "items(last)"]
for i in range(12):
    eng.fill_synthetic(q, k, v, seed=100 + i); eng.step(q, k, v); eng.sync()
    n = 64 + 8 * B
    dd = np.zeros(n, dtype=np.int64); L.pikv_debug_read(eng.h, dd.ctypes.data, n)
    t8 = dd[64:].reshape(B, 8).astype(np.float64)
    t = t8[:, :6]
    t0 = t[:, 0].min()
    ph = np.diff(t[:, :5], axis=1) / 1e3
    line = " ".join("%s max %.1f med %.1f" % (nm, ph[:, j].max(), np.median(ph[:, j])) for j, nm in enumerate(names[:4]))
    span = (t[:, 4].max() - t0) / 1e3
    sub = "pass1 %.1f sync %.1f pass2 %.1f" % (((t8[:, 6] - t8[:, 3]) / 1e3).max(), ((t8[:, 7] - t8[:, 6]) / 1e3).max(),
                                              ((t8[:, 4] - t8[:, 7]) / 1e3).max())
    print("step %d: %s | retrieve: %s | start spread %.1f us, span to last retrieve %.1f us" % (
        i, line, sub, (t[:, 0].max() - t0) / 1e3, span))
eng.close()
