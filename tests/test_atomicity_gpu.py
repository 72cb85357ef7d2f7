# SPDX-License-Identifier: Apache-2.0
"""GPU: failure atomicity and state-invalidation regressions.

* An exhausted KV page pool fails the step's insert (PIKV_ERR_OUT_OF_MEMORY)
  with no partial state: slot metadata, ring heads/live counts and the pool's
  free stack are exactly as before the failing step (pipeline.cpp:153-154;
  the header's atomicity contract, include/pikv_b200.h:17).  Both insert
  paths are covered: distinct rings (warp-parallel) and k entries sharing a
  ring (sequential), and the bulk store build.
* pikv_set_codec_host after the pinned host-graph step has been captured:
  later pinned steps must use the new basis (the graph is re-captured).
* Duo with saliency=None: per_layer_scores are empty, so the fold-back skips
  them and the Duo score is 0 (pipeline.cpp:307; scheduler.cpp:222-226).
"""
import numpy as np
import pytest

from cases import engine_config
from oracle_bind import OracleEngine, make_stream
from test_engine_gpu import run_parity, to_kv

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2508_06526_b200.engine import Engine, PikvError  # noqa: E402


def _state(eng, s):
    st = eng.slots(s)
    return {k: v.copy() for k, v in st.items()}, eng.store_stats(s), eng.pool_pages_in_use()


def _same(a, b):
    sa, ta, pa = a
    sb, tb, pb = b
    for key in sa:
        assert np.array_equal(sa[key], sb[key]), key
    assert ta == tb and pa == pb


@pytest.mark.parametrize("kw", [
    dict(E=8, n_tok=1, n_exp=8, G=1),          # k distinct rings: warp-parallel insert
    dict(E=8, n_tok=1, n_exp=2, G=1, k=4),     # experts share rings: sequential insert
])
def test_pool_exhaustion_leaves_no_partial_state(kw):
    k = kw.pop("k", 2)
    cfg = engine_config(router="TopK", unbounded=True, S=64, ps=4, batch=2, k=k, **kw)
    cfg.pool_entries = 24  # 6 pages of 4 entries for both streams together
    eng = Engine(cfg)
    B, d = 2, cfg.model.d
    streams = [make_stream(80, d, 5 + s) for s in range(B)]
    failed = False
    for t in range(80):
        before = [_state(eng, s) for s in range(B)]
        q = np.stack([streams[s][0][t] for s in range(B)])
        kk = np.stack([streams[s][1][t] for s in range(B)])
        v = np.stack([streams[s][2][t] for s in range(B)])
        eng.step_host(to_kv(q, "f32"), to_kv(kk, "f32"), to_kv(v, "f32"), None)
        _, _, _, summ = eng.read_step()
        errs = [summ[s]["error"] for s in range(B)]
        if any(errs):
            with pytest.raises(PikvError) as ei:
                eng.sync()
            assert ei.value.kind == "OutOfMemory"
            for s in range(B):
                if errs[s]:
                    # the failing stream's store is exactly as before the step
                    sa, ta, _ = _state(eng, s)
                    sb, tb, _ = before[s]
                    for key in sa:
                        assert np.array_equal(sa[key], sb[key]), (t, s, key)
                    assert ta == tb, (t, s)
            failed = True
            break
    assert failed, "the pool never ran out"
    # pages of the failed step went back: in-use pages = live pages
    assert eng.pool_pages_in_use() <= 6


def test_bulk_exhaustion_leaves_no_partial_state():
    cfg = engine_config(router="TopK", unbounded=True, d=64, S=256, ps=16, batch=1, E=8, G=1,
                        n_tok=1, n_exp=8, n_layers=0)
    cfg.pool_entries = 64  # 4 pages of 16
    eng = Engine(cfg)
    rng = np.random.default_rng(1)
    T = 60
    k = rng.standard_normal((T, 64)).astype(np.float32)
    v = rng.standard_normal((T, 64)).astype(np.float32)
    ex = np.stack([rng.choice(8, 2, replace=False) for _ in range(T)]).astype(np.int32)
    before = _state(eng, 0)
    with pytest.raises(PikvError) as ei:
        eng.insert_bulk_host(0, k, v, ex)
    assert ei.value.kind == "OutOfMemory"
    _same(_state(eng, 0), before)


def test_set_codec_after_host_graph_capture():
    """pikv_set_codec_host must drop the pinned host-step graph."""
    from paper_2508_06526_b200 import _capi
    d, H, r = 128, 2, 8
    cfg = engine_config(router="TopK", sched="LRU", d=d, H=H, S=64, batch=2, codec="LowRank",
                        rank=r, n_layers=0)
    rng = np.random.default_rng(9)
    b1, b2 = (np.ascontiguousarray(np.linalg.qr(rng.standard_normal((64, 64)))[0][:, :r].T[None]
                                   .repeat(H, 0), dtype=np.float32) for _ in range(2))
    a, b = Engine(cfg), Engine(cfg)  # a: pinned packed host graph; b: device path
    a.set_codec(b1), b.set_codec(b1)
    B, T = 2, 10
    st = [make_stream(T, d, 31 + s) for s in range(B)]
    host = torch.empty(T, 3, B, d, dtype=torch.float32).pin_memory()
    for t in range(T):
        for j in range(3):
            host[t, j] = torch.from_numpy(np.stack([st[s][j][t] for s in range(B)]).astype(np.float32))
    hy = torch.empty(B, cfg.stored_width, dtype=torch.float32).pin_memory()
    L = _capi.lib()
    for t in range(T):
        if t == 5:
            a.set_codec(b2), b.set_codec(b2)
        dev = host[t].cuda()
        yb = b.step(dev[0], dev[1], dev[2]).cpu()
        _capi.check(L.pikv_step_host(a.h, host[t, 0].data_ptr(), host[t, 1].data_ptr(),
                                     host[t, 2].data_ptr(), None, hy.data_ptr()))
        assert torch.equal(yb, hy), t


def test_duo_without_saliency_matches_oracle():
    """Duo with saliency=None: empty per-layer scores (no fold, score 0)."""
    cfg = engine_config(router="Base", sched="Duo", n_layers=5, batch=2)
    run_parity(cfg, 50, 37, no_saliency=True)
