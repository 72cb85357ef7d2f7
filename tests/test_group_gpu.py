# SPDX-License-Identifier: Apache-2.0
"""GPU: the micro-batch pipeline (pikv_group_*) changes only the schedule.

A group of n micro-batch engines is stepped without host synchronisation
(micro-batch m's control plane overlaps micro-batch m-1's attention), with
device and pinned-host submissions mixed.  Each micro-batch must produce
exactly what a standalone engine of the same streams produces when stepped
one call at a time: y bit-identical every step (same attention grid, so the
same work-item split), and the final slot metadata, router state and
scheduler state bit-identical.  The standalone engine itself is checked
against the CPU oracle in test_engine_gpu.py.
"""
import dataclasses

import numpy as np
import pytest

from cases import engine_config

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2508_06526_b200.engine import Engine, EngineGroup  # noqa: E402


def bf16_bits(x):
    f = np.ascontiguousarray(x, dtype=np.float32)
    return (f.view(np.uint32) >> 16).astype(np.uint16)


@pytest.mark.parametrize("n_micro,sched,codec", [(2, "LRU", "Identity"), (2, "H2O", "Identity"),
                                                 (4, "LRUPlus", "Identity"), (2, "LRU", "Int8"),
                                                 (2, "H2O", "Int4"), (2, "LRU", "LowRank")])
def test_group_matches_standalone_engines(monkeypatch, n_micro, sched, codec):
    monkeypatch.setenv("PIKV_ATTEND_SMS", "12")  # same attention grid for both sides
    B, T = 8, 48
    cfg = engine_config(router="TopK", sched=sched, d=256, H=4, E=8, k=2, S=64, G=2, n_tok=1,
                        n_exp=8, budget=6, ps=4, n_layers=0, dtype="bf16", batch=B, codec=codec,
                        rank=16)
    Bm = B // n_micro
    grp = EngineGroup(cfg, n_micro=n_micro, attend_sms=12)
    refs = [Engine(dataclasses.replace(cfg, batch=Bm)) for _ in range(n_micro)]
    if codec == "LowRank":
        hd = cfg.model.d // cfg.n_heads
        basis = np.linalg.qr(np.random.default_rng(1).standard_normal((hd, hd)))[0][:, :16].T
        basis = np.ascontiguousarray(np.repeat(basis[None], cfg.n_heads, 0), np.float32)
        grp.set_codec(basis)
        for r in refs:
            r.set_codec(basis)
    rng = np.random.default_rng(5)
    x = bf16_bits(rng.standard_normal((T, 3, B, cfg.model.d)))
    dev = torch.from_numpy(x.view(np.int16)).cuda()
    host = torch.from_numpy(x.view(np.int16)).pin_memory()
    dp = cfg.stored_width
    ys = torch.zeros(T, B, dp, dtype=torch.float32, device="cuda")
    hy = torch.zeros(T, B, dp, dtype=torch.float32).pin_memory()
    torch.cuda.synchronize()
    for t in range(T):
        for m in range(n_micro):
            sl = slice(m * Bm, (m + 1) * Bm)
            if t % 3 == 2:  # pinned host buffers, copied on the micro-batch's stream
                grp.submit(m, host[t, 0, sl].data_ptr(), host[t, 1, sl].data_ptr(),
                           host[t, 2, sl].data_ptr(), None, hy[t, sl].data_ptr(), host=True)
            else:
                grp.submit(m, dev[t, 0, sl].data_ptr(), dev[t, 1, sl].data_ptr(),
                           dev[t, 2, sl].data_ptr(), None, ys[t, sl].data_ptr())
    grp.sync()
    got = ys.cpu().numpy()
    got_h = hy.numpy()
    for t in range(T):
        for m in range(n_micro):
            sl = slice(m * Bm, (m + 1) * Bm)
            y = refs[m].step(dev[t, 0, sl], dev[t, 1, sl], dev[t, 2, sl])
            want = y.cpu().numpy()
            g = got_h[t, sl] if t % 3 == 2 else got[t, sl]
            assert np.array_equal(g, want), (t, m)
    for m in range(n_micro):
        e, r = grp.engines[m], refs[m]
        for s in range(Bm):
            a, b = e.slots(s), r.slots(s)
            for key in a:
                assert np.array_equal(np.asarray(a[key]), np.asarray(b[key])), (m, s, key)
            ra, rb = e.router_state(s), r.router_state(s)
            for key in ra:
                assert np.array_equal(np.asarray(ra[key]), np.asarray(rb[key])), (m, s, key)
            assert e.scheduler_state(s) == r.scheduler_state(s)
    _, _, _, summ = grp.read_step()
    assert all(s["error"] == 0 for s in summ)
    assert sum(s["n_attended"] for s in summ) > 0
    grp.close()
    for r in refs:
        r.close()


def test_group_step_full_batch_buffers():
    """pikv_group_step on full-batch device tensors == per-micro submits."""
    B, T = 4, 12
    cfg = engine_config(router="TopK", sched="LRU", d=128, H=2, E=8, k=2, S=64, G=2, n_tok=1,
                        n_exp=8, budget=6, ps=4, n_layers=0, dtype="bf16", batch=B)
    a = EngineGroup(cfg, n_micro=2)
    b = EngineGroup(cfg, n_micro=2)
    rng = np.random.default_rng(9)
    x = torch.from_numpy(bf16_bits(rng.standard_normal((T, 3, B, cfg.model.d))).view(np.int16)).cuda()
    for t in range(T):
        ya = a.step(x[t, 0], x[t, 1], x[t, 2])
        yb = torch.empty_like(ya)
        for m in range(2):
            sl = slice(2 * m, 2 * m + 2)
            b.submit(m, x[t, 0, sl].data_ptr(), x[t, 1, sl].data_ptr(), x[t, 2, sl].data_ptr(), None,
                     yb[sl].data_ptr())
        b.sync()
        assert torch.equal(ya, yb)
    a.close()
    b.close()


@pytest.mark.parametrize("n_micro", [2, 4])
def test_attention_partition_changes_only_the_schedule(monkeypatch, n_micro):
    """The attention SM partition (green context; launches of different
    micro-batches unordered and overlapping) against the ordered pipeline on
    all SMs, same attention grid (104 SMs, a multiple of 8): y, experts and
    attended counts bit-identical every step at the c2 head shape (32 x 128
    bf16, E16 top-2); the partition is reported active only when asked for."""
    B, T, d = 8, 12, 4096
    cfg = engine_config(router="TopK", sched="LRU", d=d, H=32, E=16, k=2, S=64, G=1, n_tok=1,
                        n_exp=16, budget=6, ps=16, n_layers=0, dtype="bf16", batch=B)
    cfg.model.head_width = 128
    rng = np.random.default_rng(9)
    x = torch.from_numpy(bf16_bits(rng.standard_normal((T, 3, B, d))).view(np.int16)).cuda()
    out = []
    for green in ("1", "0"):
        monkeypatch.setenv("PIKV_GREEN", green)
        grp = EngineGroup(cfg, n_micro=n_micro, attend_sms=104)
        assert grp.attention_partition() == (green == "1")
        Bm = B // n_micro
        ys = torch.zeros(T, B, cfg.stored_width, dtype=torch.float32, device="cuda")
        rec = []
        for t in range(T):
            for m in range(n_micro):
                sl = slice(m * Bm, (m + 1) * Bm)
                grp.submit(m, x[t, 0, sl], x[t, 1, sl], x[t, 2, sl], None, ys[t, sl])
            grp.sync()
            steps = [e.read_step() for e in grp.engines]
            rec.append((np.concatenate([s[0] for s in steps]),
                        [x_["n_attended"] for s in steps for x_ in s[3]]))
        out.append((ys.cpu().numpy(), rec))
        grp.close()
    (y1, r1), (y0, r0) = out
    assert np.array_equal(y1.view(np.uint32), y0.view(np.uint32))
    for t in range(T):
        assert np.array_equal(r1[t][0], r0[t][0]) and r1[t][1] == r0[t][1], t
