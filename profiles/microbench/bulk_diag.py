import ctypes, os, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from bench import make_config, WORKLOADS
from paper_2508_06526_b200.engine import Engine
from paper_2508_06526_b200 import _capi
for T in (8192, 32768):
    w = dict(WORKLOADS["c4-lowrank"][1]); w["B"] = 2; w["codec"] = "Identity"
    cfg = make_config(w); cfg.pool_entries = 4 * T * cfg.router.k + 65536
    t0 = time.perf_counter(); eng = Engine(cfg); print("create", time.perf_counter() - t0)
    d = w["H"] * w["hd"]
    k = torch.randn(T, d, device="cuda").to(torch.bfloat16); v = torch.randn(T, d, device="cuda").to(torch.bfloat16)
    ex = torch.stack([torch.randperm(cfg.model.E, device="cuda")[:cfg.router.k] for _ in range(T)]).int()
    L = _capi.lib(); nd = ctypes.c_int64(0)
    for rep in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        _capi.check(L.pikv_insert_bulk(eng.h, rep % 2, T, k.data_ptr(), v.data_ptr(), ex.data_ptr(), None, ctypes.byref(nd)))
        t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
        print(T, rep, "call %.2f ms, sync %.2f ms" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3))
    eng.close()
