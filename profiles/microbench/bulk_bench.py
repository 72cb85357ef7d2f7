"""Bulk store build (pikv_insert_bulk) timing: T tokens into one stream of
a c4-lowrank-shaped engine (32 heads x 128 -> rank 32, bf16) with the
projection on tcgen05 (PIKV_BULK_TC=1) or CUDA cores (=0); also identity.
Prints one JSON line per variant: ms, tokens/s, KV bytes in/out."""
import ctypes, json, os, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from bench import make_config, WORKLOADS
from paper_2508_06526_b200.engine import Engine
from paper_2508_06526_b200 import _capi

T = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
for codec in ("LowRank", "Identity"):
    for tc in (("1", "0") if codec == "LowRank" else ("1",)):
        os.environ["PIKV_BULK_TC"] = tc
        w = dict(WORKLOADS["c4-lowrank"][1]); w["B"] = 2; w["codec"] = codec
        cfg = make_config(w)
        cfg.pool_entries = 4 * T * cfg.router.k + 65536
        eng = Engine(cfg)
        hd, r, H, d = w["hd"], w.get("rank", 32), w["H"], w["H"] * w["hd"]
        if codec == "LowRank":
            basis = np.linalg.qr(np.random.default_rng(0).standard_normal((hd, hd)))[0][:, :r].T
            eng.set_codec(np.ascontiguousarray(np.repeat(basis[None], H, 0), np.float32))
        k = torch.randn(T, d, device="cuda").to(torch.bfloat16)
        v = torch.randn(T, d, device="cuda").to(torch.bfloat16)
        ex = torch.stack([torch.randperm(cfg.model.E, device="cuda")[:cfg.router.k] for _ in range(T)]).int()
        L = _capi.lib(); nd = ctypes.c_int64(0)
        res = []
        for rep in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            _capi.check(L.pikv_insert_bulk(eng.h, rep % 2, T, k.data_ptr(), v.data_ptr(), ex.data_ptr(), None,
                                           ctypes.byref(nd)))
            torch.cuda.synchronize(); res.append(time.perf_counter() - t0)
        ms = min(res[1:]) * 1e3
        print(json.dumps({"codec": codec, "tensor_cores": tc == "1", "tokens": T, "ms": ms,
                          "tokens_per_s": T / ms * 1e3, "kv_in_gb": 2 * T * d * 2 / 1e9,
                          "entries": T * cfg.router.k, "entry_bytes": eng.entry_bytes()}))
        eng.close()
