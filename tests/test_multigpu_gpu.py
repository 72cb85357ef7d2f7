# SPDX-License-Identifier: Apache-2.0
"""The sharded (multi-GPU) step on one B200.

* NCCL inside the library: an engine with a one-rank NCCL communicator runs
  the exchange path -- combine into the exchange record, ncclAllGather on the
  engine stream inside the captured step graph, the cross-rank LSE merge --
  and must equal the plain single-rank step (routing, evictions and store
  bit-exact; y within 1e-6).  Same for the micro-batch group (one
  communicator per micro-batch).
* Two processes driving real CUDA engines of world_size 2 (rank r owns the
  logical devices g % 2 == r, kvstore.cpp:14-30 placement) through
  pikv_step_local / all-gather / pikv_step_finish, the all-gather staged
  through host memory by gloo (two ranks cannot share a GPU in one NCCL
  communicator, so this is the one-GPU rehearsal of the 8-GPU exchange):
  every rank's y, experts and hits equal the CPU oracle's single-store
  step, and the union of the ranks' eviction records is the oracle's.
"""
import os
import socket

import numpy as np
import pytest

from cases import engine_config
from oracle_bind import OracleEngine, make_stream

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2508_06526_b200.engine import Engine, EngineGroup  # noqa: E402
from test_engine_gpu import rel_l2, to_kv  # noqa: E402


def _inputs(cfg, T, seed):
    B, d = cfg.batch, cfg.model.d
    st = [make_stream(T, d, seed + 100 * s, cfg.kv_dtype, 0) for s in range(B)]
    out = []
    for t in range(T):
        out.append([torch.from_numpy(to_kv(np.stack([st[s][j][t] for s in range(B)]), cfg.kv_dtype)
                                     .view(np.int16 if cfg.kv_dtype == "bf16" else np.float32)).cuda()
                    for j in range(3)])
    return out, st


@pytest.mark.parametrize("sched", ["LRU", "H2O"])
def test_one_rank_nccl_exchange_path(sched):
    cfg = engine_config(router="TopK", sched=sched, d=256, H=4, S=64, batch=3, dtype="bf16",
                        G=2, n_tok=1, n_exp=8, budget=3, n_layers=0)
    a, b = Engine(cfg), Engine(cfg)
    b.attach_nccl(Engine.nccl_unique_id())  # world 1: a one-rank communicator
    ins, _ = _inputs(cfg, 30, 5)
    for t, (q, k, v) in enumerate(ins):
        ya = a.step(q.view(torch.bfloat16), k.view(torch.bfloat16), v.view(torch.bfloat16)).cpu().numpy()
        yb = b.step(q.view(torch.bfloat16), k.view(torch.bfloat16), v.view(torch.bfloat16)).cpu().numpy()
        ea, ga, _, sa = a.read_step()
        eb, gb, _, sb = b.read_step()
        assert np.array_equal(ea, eb) and np.array_equal(ga, gb), t
        assert [(x["hits"], x["n_attended"], x["pages_after"]) for x in sa] == \
               [(x["hits"], x["n_attended"], x["pages_after"]) for x in sb], t
        assert a.read_evictions() == b.read_evictions(), t
        for s in range(cfg.batch):
            assert rel_l2(yb[s].astype(np.float64), ya[s].astype(np.float64)) <= 1e-6, (t, s)
    for s in range(cfg.batch):
        sa_, sb_ = a.slots(s), b.slots(s)
        assert np.array_equal(sa_["id"], sb_["id"])
        live = sa_["id"] != 0  # (never-written slots hold uninitialised values)
        for key in ("token", "expert", "freq", "last_access"):
            assert np.array_equal(sa_[key][live], sb_[key][live]), key
        assert np.allclose(sa_["attn_mass"][live], sb_["attn_mass"][live], rtol=1e-5, atol=1e-7)


def test_one_rank_nccl_group():
    cfg = engine_config(router="TopK", sched="LRU", d=256, H=4, S=64, batch=4, dtype="bf16",
                        G=2, n_tok=1, n_exp=8, budget=3, n_layers=0)
    ga, gb = EngineGroup(cfg, n_micro=2), EngineGroup(cfg, n_micro=2)
    gb.attach_nccl([Engine.nccl_unique_id() for _ in range(2)])
    ins, _ = _inputs(cfg, 20, 9)
    for t, (q, k, v) in enumerate(ins):
        bq, bk, bv = (x.view(torch.bfloat16) for x in (q, k, v))
        ya = ga.step(bq, bk, bv)
        yb = gb.step(bq, bk, bv)
        torch.cuda.synchronize()
        assert torch.allclose(ya, yb, rtol=1e-5, atol=1e-6), t
        assert np.array_equal(ga.read_step()[0], gb.read_step()[0]), t
    # pinned host submits: the sharded host path copies y out right after the
    # cross-rank merge (an event inside the fold graph)
    Bm = cfg.batch // 2
    hin = torch.empty(6, 2, 3, Bm, cfg.model.d, dtype=torch.int16).pin_memory()
    for t in range(6):
        q, k, v = ins[t]
        for m in range(2):
            for j, x in enumerate((q, k, v)):
                hin[t, m, j] = x[m * Bm:(m + 1) * Bm].cpu()
    hya = torch.zeros(6, cfg.batch, cfg.stored_width).pin_memory()
    hyb = torch.zeros(6, cfg.batch, cfg.stored_width).pin_memory()
    for t in range(6):
        for m in range(2):
            for g, hy in ((ga, hya), (gb, hyb)):
                g.submit(m, hin[t, m, 0].data_ptr(), hin[t, m, 1].data_ptr(), hin[t, m, 2].data_ptr(), None,
                         hy[t, m * Bm].data_ptr(), host=True)
    ga.sync(), gb.sync()
    assert torch.allclose(hya, hyb, rtol=1e-5, atol=1e-6)
    assert hyb.abs().sum() > 0
    ga.close(), gb.close()


# ------------------------------------------------ two ranks, one GPU ----
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, T, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_06526_b200.parallel import ShardedStepper
    cfg = _two_rank_cfg()
    cfg.world_size, cfg.rank_id = world, rank
    eng = Engine(cfg)
    stepper = ShardedStepper(eng)
    ins, _ = _inputs(cfg, T, 21)
    ys, experts, summ, evs = [], [], [], []
    for q, k, v in ins:
        y = stepper.step(q.view(torch.bfloat16), k.view(torch.bfloat16), v.view(torch.bfloat16))
        torch.cuda.synchronize()
        ys.append(y.cpu().numpy())
        e, _, _, sm = eng.read_step()
        experts.append(e)
        summ.append([(x["hits"], x["lookups"], x["n_attended"]) for x in sm])
        why = {"budget": 0, "threshold": 1, "overwrite": 2}
        evs.append([(r.stream, r.step, r.entry_id, r.token_id, r.expert_id, r.device, why[r.reason])
                    for r in eng.read_evictions()])
    np.save(os.path.join(out_dir, "rank%d.npy" % rank),
            np.array({"y": ys, "experts": experts, "summ": summ, "evs": evs,
                      "local": eng.local_attended()}, dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()
    eng.close()


def _two_rank_cfg():
    return engine_config(router="TopK", sched="LRU", d=256, H=4, S=64, batch=2, dtype="bf16",
                         G=2, n_tok=1, n_exp=8, budget=3, n_layers=0)


def test_two_process_sharded_step_matches_oracle(tmp_path):
    import torch.multiprocessing as mp
    T, world = 25, 2
    mp.start_processes(_rank_main, args=(world, _free_port(), T, str(tmp_path)), nprocs=world,
                       start_method="spawn")
    res = [np.load(tmp_path / ("rank%d.npy" % r), allow_pickle=True).item() for r in range(world)]
    cfg = _two_rank_cfg()
    _, st = _inputs(cfg, T, 21)
    orc = [OracleEngine(cfg) for _ in range(cfg.batch)]
    for t in range(T):
        for s in range(cfg.batch):
            r = orc[s].step(st[s][0][t], st[s][1][t], st[s][2][t])
            for rk in range(world):
                assert res[rk]["experts"][t][s].tolist() == r["experts"], (t, s, rk)
                hits, lookups, n_att = res[rk]["summ"][t][s]
                assert (hits, lookups, n_att) == (r["hits"], r["lookups"], r["n_attended"]), (t, s, rk)
                assert rel_l2(res[rk]["y"][t][s].astype(np.float64), r["y"]) <= 2e-5, (t, s, rk)
            # rank r evicts its own devices (g % 2 == r): the union is the oracle's
            mine = sorted((e[1], e[2], e[3], e[4], e[5], e[6]) for rk in range(world)
                          for e in res[rk]["evs"][t] if e[0] == s)
            want = sorted((e[0], e[1], e[2], e[3], e[4], e[6]) for e in r["evictions"])
            assert mine == want, (t, s)
    # each rank attended only its own shards: the two local counts add up
    assert res[0]["local"] + res[1]["local"] == sum(res[0]["summ"][-1][s][2] for s in range(cfg.batch))
