"""Per-CTA anatomy of one k_attend launch inside the micro-batch pipeline
(PIKV_DEBUG_ATT=1: each CTA's consumer thread 0 stamps globaltimer at start
and exit, its item and entry counts and its SM id): start skew, finish
spread (the launch's tail), CTAs per SM and per-CTA throughput.

    python profiles/microbench/attend_ctas.py [--config c2] [--micro 2]
"""
import argparse
import ctypes
import os
import sys

os.environ["PIKV_DEBUG_ATT"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_06526_b200._capi import lib  # noqa: E402
from paper_2508_06526_b200.engine import EngineGroup  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--micro", type=int, default=2)
ap.add_argument("--attend-sms", type=int, default=None)
ap.add_argument("--steps", type=int, default=12)
args = ap.parse_args()

w = bench.WORKLOADS[args.config][1]
cfg = bench.make_config(w)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
sms = args.attend_sms or (nsm - {"Int8": 12, "Int4": 24}.get(w["codec"], 44) if args.micro > 1 else nsm)
grp = EngineGroup(cfg, n_micro=args.micro, attend_sms=sms, device=0)
if cfg.compressor.scheme in ("LowRank",):
    hd, r = cfg.head_dim, cfg.compressor.rank
    basis = np.linalg.qr(np.random.default_rng(0).standard_normal((hd, hd)))[0][:, :r].T
    grp.set_codec(np.ascontiguousarray(np.repeat(basis[None], cfg.n_heads, 0), np.float32))
grp.prefill_synthetic(w["L"], seed=7)
tdt = torch.bfloat16 if cfg.kv_dtype == "bf16" else torch.float32
Bm, d, n = grp.Bm, cfg.model.d, args.micro
q = torch.randn(n, 3, Bm, d, device="cuda").to(tdt)
y = torch.empty(cfg.batch, cfg.stored_width, dtype=torch.float32, device="cuda")
L = lib()
L.pikv_debug_read.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong), ctypes.c_int]
e0 = grp.engines[0]
tc = os.environ.get("PIKV_BF16TC") == "1"  # the HMMA kernel: one CTA per SM, wait ns in slot 6
ctas = (1 if tc else 3 if os.environ.get("PIKV_ATT_CPS") == "3" else 2) * sms
nbuf = 64 + 8 * Bm + 8 * ctas
buf = (ctypes.c_longlong * nbuf)()
eb = e0.entry_bytes()
res = []
for i in range(args.steps):
    for m in range(n):
        grp.submit(m, q[m, 0].data_ptr(), q[m, 1].data_ptr(), q[m, 2].data_ptr(), None,
                   y[m * Bm:(m + 1) * Bm].data_ptr())
    grp.sync()
    if i < 3:
        continue
    L.pikv_debug_read(e0.h, buf, nbuf)
    a = np.array(buf[64 + 8 * Bm:], dtype=np.int64).reshape(ctas, 8)
    t0, t1, items, ents, sm = a[:, 0], a[:, 1], a[:, 2], a[:, 3], a[:, 4]
    te, tf = a[:, 5], a[:, 6]
    wait = a[:, 6] if tc else a[:, 7]
    if tc:
        tf = te
    base = te.min()
    start, end = (t0 - base) / 1e3, (t1 - base) / 1e3
    per_sm = np.bincount(sm, minlength=nsm)
    dur = end.max()
    gbs = ents.sum() * eb / (dur * 1e-6) / 1e9
    rate = ents * eb / np.maximum(end - start, 1e-3) / 1e3  # GB/s per CTA
    two = per_sm[sm] >= 2
    res.append(dict(wait_frac_p50=np.percentile(wait / np.maximum(t1 - t0, 1), 50), entry_max=((te - base) / 1e3).max(), setup_p50=np.percentile((t0 - te) / 1e3, 50),
                    first_data_p50=np.percentile((tf - base) / 1e3, 50),
                    first_data_max=((tf - base) / 1e3).max(), launch_us=dur, gbs=gbs, start_max=start.max(), end_min=end.min(),
                    end_p50=np.percentile(end, 50), items_min=items.min(), items_max=items.max(),
                    sms_used=int((per_sm > 0).sum()), sms_with_2=int((per_sm >= 2).sum()),
                    rate_alone=rate[~two].mean() if (~two).any() else 0.0,
                    rate_paired=rate[two].mean() if two.any() else 0.0))
keys = list(res[0])
print(f"{args.config} micro={n} attend_sms={sms} ctas={ctas} entry={eb} B")
for k in keys:
    v = np.array([r[k] for r in res], dtype=np.float64)
    print(f"  {k:12s} mean {v.mean():9.2f}  min {v.min():9.2f}  max {v.max():9.2f}")
