"""Timeline of the micro-batch pipeline (pikv_group) at a bench workload:
per submit, CUDA events before / after the control graph, after the cross-
micro-batch wait, after the attention graph and after the tail graph
(PIKV_GROUP_TIMELINE=1, pikv_group_read_timeline).  Prints the mean phase
lengths, the gap between one micro-batch's attention end and the next one's
start, and whether that next attention waited on its own control plane
(slack < 0) or on the event hand-off.

    python profiles/microbench/group_timeline.py [--config c2] [--steps 40]
"""
import argparse
import ctypes
import os
import sys

os.environ["PIKV_GROUP_TIMELINE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_06526_b200._capi import check, lib  # noqa: E402
from paper_2508_06526_b200.engine import EngineGroup  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--attend-sms", type=int, default=None)
ap.add_argument("--micro", type=int, default=2)
ap.add_argument("--bank", action="store_true", help="distinct q/k/v per step (as bench.py)")
ap.add_argument("--copy", action="store_true", help="stage each step's q/k/v with a D2D copy (as bench.py)")
args = ap.parse_args()

w = bench.WORKLOADS[args.config][1]
cfg = bench.make_config(w)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
sms = args.attend_sms or nsm - {"Int8": 12, "Int4": 24}.get(w["codec"], 44)
grp = EngineGroup(cfg, n_micro=args.micro, attend_sms=sms, device=0)
if cfg.compressor.scheme in ("LowRank",):
    hd, r = cfg.head_dim, cfg.compressor.rank
    basis = np.linalg.qr(np.random.default_rng(0).standard_normal((hd, hd)))[0][:, :r].T
    grp.set_codec(np.ascontiguousarray(np.repeat(basis[None], cfg.n_heads, 0), np.float32))
grp.prefill_synthetic(w["L"], seed=7)
tdt = torch.bfloat16 if cfg.kv_dtype == "bf16" else torch.float32
Bm, d, n = grp.Bm, cfg.model.d, args.micro
q = torch.randn(n, 3, Bm, d, device="cuda").to(tdt)
nb = 5 + args.steps
bank = torch.randn(nb if args.bank else 1, n, 3, Bm, d, device="cuda").to(tdt)
streams = [e.external_stream() for e in grp.engines]
it = [0]
y = torch.empty(cfg.batch, cfg.stored_width, dtype=torch.float32, device="cuda")


def step():
    i = it[0] % bank.shape[0]
    it[0] += 1
    for m in range(n):
        src = bank[i, m]
        if args.copy:
            with torch.cuda.stream(streams[m]):
                q[m].copy_(src, non_blocking=True)
            src = q[m]
        grp.submit(m, src[0].data_ptr(), src[1].data_ptr(), src[2].data_ptr(), None,
                   y[m * Bm:(m + 1) * Bm].data_ptr())


for _ in range(5):
    step()
grp.sync()
buf = (ctypes.c_double * (6 * 4096))()
cnt = ctypes.c_int32()
check(lib().pikv_group_read_timeline(grp.h, buf, 4096, ctypes.byref(cnt)))  # drop warm-up rows
print('warm-up rows', cnt.value)
for _ in range(args.steps):
    step()
grp.sync()
check(lib().pikv_group_read_timeline(grp.h, buf, 4096, ctypes.byref(cnt)))
print('rows', cnt.value)
rows = np.frombuffer(buf, dtype=np.float64)[:6 * cnt.value].reshape(-1, 6)
m, c0, c1, a0, a1, t1 = rows.T
order = np.argsort(a0)
r = rows[order][n:]  # skip the first step
ctl = (r[:, 2] - r[:, 1]) * 1e3
att = (r[:, 4] - r[:, 3]) * 1e3
tail = (r[:, 5] - r[:, 4]) * 1e3
# gap: this attention's start (wait satisfied) minus the previous attention's end
prev_end = rows[order][n - 1:-1, 4]
gap = (r[:, 3] - prev_end) * 1e3
# slack: previous attention end minus this micro-batch's control end (> 0: control was ready)
slack = (prev_end - r[:, 2]) * 1e3
step_ms = (r[-1, 4] - r[0, 4]) / (len(r) - 1) * n
print(f"{args.config} attend_sms={sms} micro={n}: step {step_ms:.4f} ms")
for k, v in [("control graph (us)", ctl), ("attention graph (us)", att), ("tail graph (us)", tail),
             ("attention gap (us)", gap), ("control slack (us)", slack)]:
    print(f"  {k:22s} mean {v.mean():7.1f}  p10 {np.percentile(v, 10):7.1f}  p90 {np.percentile(v, 90):7.1f}")
print("  attention share of timeline: %.3f" % (att.sum() / ((r[-1, 4] - r[0, 3]) * 1e3)))
