# SPDX-License-Identifier: Apache-2.0
"""The store build of a prefill: pikv_insert_bulk vs the
oracle's T x k sequential inserts (po_engine_insert_bulk).

Bit-exact: displacement count, every slot's metadata (ids, shard_seq,
tokens, experts, steps, freq), store totals, the snapshot; then decode
steps run on both and must agree (evictions bit-exact -- the rebuilt page
records and live-page counters are right -- and y within the tolerance of
test_engine_gpu.py, which checks the bulk-written payloads through every
codec)."""
import numpy as np
import pytest

from cases import engine_config
from oracle_bind import OracleEngine, make_stream

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2508_06526_b200.engine import Engine  # noqa: E402
from test_engine_gpu import Y_TOL, rel_l2, to_kv  # noqa: E402


def codec_params(codec, d, H, rank, rng):
    hd = d // H
    basis = bias = kept = None
    if codec in ("LowRank", "LoRAPlus"):
        basis = np.linalg.qr(rng.standard_normal((hd, hd)))[0][:, :rank].T[None].repeat(H, 0)
        basis = np.ascontiguousarray(basis, dtype=np.float32)
        if codec == "LoRAPlus":
            bias = (0.1 * rng.standard_normal(d)).astype(np.float32).astype(np.float64)
    if codec == "Prune":
        kept = np.stack([np.sort(rng.choice(hd, rank, replace=False)) for _ in range(H)]).astype(np.int32)
    return basis, bias, kept


def compare_state(eng, orc, B, T_now):
    for s in range(B):
        a, b = eng.slots(s), orc[s].slots()
        assert np.array_equal(a["id"], b["id"]), s
        live = a["id"] != 0
        for key in ("shard_seq", "token", "expert", "insert_step", "last_access", "freq"):
            assert np.array_equal(a[key][live], b[key][live]), (s, key)
        assert eng.store_stats(s) == orc[s].store_stats(), s
        assert np.array_equal(eng.snapshot(s), orc[s].snapshot(T_now[s]))


@pytest.mark.parametrize("codec,dtype,kw", [
    ("Identity", "f32", dict(S=16, ps=4, budget=3)),      # rings overwrite inside the bulk
    ("Identity", "bf16", dict(S=64, H=2, n_layers=3)),
    ("Int8", "f32", dict(S=32, H=2)),
    ("Int4", "bf16", dict(S=32, H=2)),
    ("LowRank", "bf16", dict(S=32, H=2)),
    ("LoRAPlus", "f32", dict(S=32, H=2)),
    ("Prune", "f32", dict(S=32, H=2)),
])
def test_insert_bulk_matches_sequential_inserts(codec, dtype, kw):
    d, rank, B = 64, 8, 3
    rng = np.random.default_rng(11)
    cfg = engine_config(router="TopK", sched="LRU", d=d, batch=B, codec=codec, rank=rank,
                        dtype=dtype, **kw)
    H = cfg.n_heads
    basis, bias, kept = codec_params(codec, d, H, rank, rng)
    eng = Engine(cfg)
    if basis is not None or kept is not None:
        eng.set_codec(basis, None if bias is None else bias.astype(np.float32), kept)
    ob = None if basis is None else np.asarray(basis, dtype=np.float64)
    orc = [OracleEngine(cfg, basis=ob, bias=bias, kept=kept) for _ in range(B)]
    nl = cfg.n_layers
    streams = [make_stream(60, d, 100 + s, dtype, nl) for s in range(B)]
    now = [0] * B

    def decode(t0, t1):
        for t in range(t0, t1):
            q = np.stack([streams[s][0][t] for s in range(B)])
            k = np.stack([streams[s][1][t] for s in range(B)])
            v = np.stack([streams[s][2][t] for s in range(B)])
            sal = None if nl == 0 else np.stack([streams[s][3][t] for s in range(B)])
            y = eng.step_host(to_kv(q, dtype), to_kv(k, dtype), to_kv(v, dtype), sal)
            evs = eng.read_evictions()
            for s in range(B):
                r = orc[s].step(q[s], k[s], v[s], None if sal is None else sal[s])
                mine = [(e.step, e.entry_id, e.token_id, e.expert_id, e.device, e.score,
                         {"budget": 0, "threshold": 1, "overwrite": 2}[e.reason])
                        for e in evs if e.stream == s]
                assert mine == r["evictions"], (t, s)
                assert rel_l2(y[s].astype(np.float64), r["y"]) <= Y_TOL, (t, s)
                now[s] += 1

    decode(0, 10)
    # bulk-build 40 tokens into stream 1 (k distinct experts per token)
    T, kk, E = 40, cfg.router.k, cfg.model.E
    experts = np.stack([rng.choice(E, kk, replace=False) for _ in range(T)]).astype(np.int32)
    bk = np.stack([streams[1][1][10 + (t % 50)] for t in range(T)])
    bv = np.stack([streams[1][2][10 + ((t + 7) % 50)] for t in range(T)])
    sal = None if nl == 0 else np.abs(rng.standard_normal((T, nl)))
    nd = eng.insert_bulk_host(1, to_kv(bk, dtype), to_kv(bv, dtype), experts, sal)
    assert nd == orc[1].insert_bulk(bk, bv, experts, sal)
    now[1] += T
    compare_state(eng, orc, B, now)
    decode(10, 30)   # decode on top: the LRU budget cuts the bulk-built pages
    compare_state(eng, orc, B, now)


def test_insert_bulk_empty_and_errors():
    cfg = engine_config(router="TopK", sched="LRU", batch=2)
    eng = Engine(cfg)
    assert eng.insert_bulk_host(0, np.zeros((0, 16), np.float32), np.zeros((0, 16), np.float32),
                                np.zeros((0, 2), np.int32)) == 0
    from paper_2508_06526_b200.engine import PikvError
    with pytest.raises(PikvError):
        eng.insert_bulk_host(5, np.zeros((1, 16), np.float32), np.zeros((1, 16), np.float32),
                             np.zeros((1, 2), np.int32))


@pytest.mark.parametrize("codec,dtype,d,H,rank", [
    ("LowRank", "bf16", 256, 2, 32),    # head width 128, bf16: the pipelined persistent kernel
    ("LoRAPlus", "bf16", 256, 2, 16),
    ("LowRank", "bf16", 128, 2, 32),
    ("LoRAPlus", "f32", 64, 2, 8),
    ("LowRank", "f32", 256, 2, 64),
])
def test_bulk_projection_tensor_cores_match_cuda_cores(monkeypatch, codec, dtype, d, H, rank):
    """The bulk projection GEMM on tcgen05 (PIKV_BULK_TC=2: tensor cores
    required, fails loudly otherwise) vs the CUDA-core fp32 projection
    (PIKV_BULK_TC=0): identical store metadata, and the decode outputs over
    the bulk-built entries agree to fp32 level (bf16 hi+lo operand split)."""
    rng = np.random.default_rng(5)
    outs = []
    for tc in ("2", "0"):
        monkeypatch.setenv("PIKV_BULK_TC", tc)
        cfg = engine_config(router="TopK", sched="LRU", unbounded=True, d=d, H=H, S=256, batch=1,
                            codec=codec, rank=rank, dtype=dtype)
        basis, bias, _ = codec_params(codec, d, H, rank, np.random.default_rng(9))
        eng = Engine(cfg)
        eng.set_codec(basis, None if bias is None else bias.astype(np.float32), None)
        T = 300
        st = make_stream(T + 4, d, 21, dtype, 0)
        ex = np.stack([np.random.default_rng(t).choice(cfg.model.E, cfg.router.k, replace=False)
                       for t in range(T)]).astype(np.int32)
        eng.insert_bulk_host(0, to_kv(st[1][:T], dtype), to_kv(st[2][:T], dtype), ex)
        ys = [eng.step_host(to_kv(st[0][T + i:T + i + 1], dtype), to_kv(st[1][T + i:T + i + 1], dtype),
                            to_kv(st[2][T + i:T + i + 1], dtype)) for i in range(4)]
        outs.append((eng.slots(0), np.concatenate(ys)))
        eng.close()
    (sa, ya), (sb, yb) = outs
    assert np.array_equal(sa["id"], sb["id"]) and np.array_equal(sa["token"], sb["token"])
    tol = 2e-3 if dtype == "bf16" else 1e-5
    assert rel_l2(ya.astype(np.float64), yb.astype(np.float64)) <= tol


@pytest.mark.parametrize("codec,d,H,rank,T", [("LowRank", 256, 2, 32, 300), ("LowRank", 4096, 32, 32, 2000),
                                               ("LowRank", 4096, 32, 16, 700), ("LoRAPlus", 256, 2, 32, 300),
                                               ("LowRank", 256, 2, 64, 260)])
def test_bulk_projection_tma_matches_register_staged(monkeypatch, codec, d, H, rank, T):
    """The TMA-fed tcgen05 projection (A tiles by cp.async.bulk.tensor into
    SWIZZLE_128B stages; by default its epilogue rounds each row to bf16 and
    writes it straight into the token's pool entries, LoRAPlus bias subtracted
    first) issues the same MMAs in the same order as the
    register-staged kernel (PIKV_BULK_TMA=0), so decode over the bulk-built
    store is bit-identical; d = 32 x 128 gives every CTA several tiles (the
    persistent loop, both ring stages) and a partial last tile."""
    rng = np.random.default_rng(11)
    outs = []
    for tma in ("1", "0"):
        monkeypatch.setenv("PIKV_BULK_TC", "2")
        monkeypatch.setenv("PIKV_BULK_TMA", tma)
        cfg = engine_config(router="TopK", sched="LRU", unbounded=True, d=d, H=H, S=4096, batch=1,
                            codec=codec, rank=rank, dtype="bf16", n_layers=0)
        basis, bias, _ = codec_params(codec, d, H, rank, np.random.default_rng(3))
        eng = Engine(cfg)
        eng.set_codec(basis, None if bias is None else bias.astype(np.float32), None)
        st = make_stream(T + 3, d, 31, "bf16", 0)
        ex = np.stack([rng.choice(cfg.model.E, cfg.router.k, replace=False) for _ in range(T)]).astype(np.int32)
        eng.insert_bulk_host(0, to_kv(st[1][:T], "bf16"), to_kv(st[2][:T], "bf16"), ex)
        ys = [eng.step_host(to_kv(st[0][T + i:T + i + 1], "bf16"), to_kv(st[1][T + i:T + i + 1], "bf16"),
                            to_kv(st[2][T + i:T + i + 1], "bf16")) for i in range(3)]
        outs.append(np.concatenate(ys))
        eng.close()
        rng = np.random.default_rng(11)
    assert np.array_equal(outs[0], outs[1])
