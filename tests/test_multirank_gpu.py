# SPDX-License-Identifier: Apache-2.0
"""The expert-sharded (world > 1) step on one GPU: two rank engines in one
process (world_size=2, G=2: logical device g lives on rank g), run as
step_local -> gather of the exchange records -> step_finish, compared with the
single-process oracle of the same G=2 store.  No kernel waits on another rank
(the gather is a host-ordered copy), so this is safe on a single GPU.

Checked per step and stream: routing, global hits/lookups/n_attended/
fetch/pages (bit-exact), y (rel-L2 <= 2e-5), each rank's scheduled eviction
records == the oracle's records of that device (in order), overwrite records
as a multiset, the attended (token, expert) union, and final slot state per
device."""
import numpy as np
import pytest

from cases import engine_config
from oracle_bind import OracleEngine, make_stream

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2508_06526_b200.engine import Engine  # noqa: E402
from paper_2508_06526_b200.parallel import device_view  # noqa: E402

REASON = {"budget": 0, "threshold": 1, "overwrite": 2}


def rel_l2(a, b):
    n = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (n if n > 0 else 1.0)


@pytest.mark.parametrize("sched,n_tok", [("LRU", 1), ("LRU", 16), ("H2O", 16), ("Duo", 1),
                                         ("AdaKV", 16)])
def test_two_rank_sharded_step_matches_oracle(sched, n_tok):
    B, T, W = 2, 60, 2
    cfg = engine_config(router="TopK", sched=sched, batch=B, G=2, n_tok=n_tok, n_exp=8, S=64,
                        H=2, budget=3, ps=4, theta0=0.05)
    ranks = []
    for r in range(W):
        c = cfg.copy()
        c.world_size, c.rank_id = W, r
        ranks.append(Engine(c))
    orc = [OracleEngine(cfg) for _ in range(B)]
    streams = [make_stream(T, 16, 300 + s, "f32", cfg.n_layers) for s in range(B)]
    nbytes = ranks[0].exchange_bytes()
    gathered = torch.empty(W * nbytes, dtype=torch.uint8, device="cuda")
    n_dev_slots = ranks[0].slots(0)["id"].size  # SPD * S per rank (one device each)
    for t in range(T):
        # inject the oracle's attn_mass / per_layer (H2O/AdaKV/Duo step-locality)
        for s in range(B):
            st = orc[s].slots()
            for r in range(W):
                sl = slice(r * n_dev_slots, (r + 1) * n_dev_slots)
                pl = st["per_layer"].reshape(-1, max(cfg.n_layers, 1))[sl].ravel()
                ranks[r].set_attn_mass(s, st["attn_mass"][sl], pl if cfg.n_layers else None)
        q = torch.tensor(np.stack([streams[s][0][t] for s in range(B)]), dtype=torch.float32, device="cuda")
        k = torch.tensor(np.stack([streams[s][1][t] for s in range(B)]), dtype=torch.float32, device="cuda")
        v = torch.tensor(np.stack([streams[s][2][t] for s in range(B)]), dtype=torch.float32, device="cuda")
        sal = torch.tensor(np.stack([streams[s][3][t] for s in range(B)]), dtype=torch.float64, device="cuda")
        ptrs = [eng.step_local(q, k, v, sal) for eng in ranks]
        for eng in ranks:
            eng.sync()
        for r in range(W):
            gathered[r * nbytes:(r + 1) * nbytes].copy_(device_view(ptrs[r], nbytes))
        torch.cuda.synchronize()
        ys = [eng.step_finish(gathered) for eng in ranks]
        for eng in ranks:
            eng.sync()
        torch.cuda.synchronize()
        reads = [eng.read_step() for eng in ranks]
        evs = [eng.read_evictions() for eng in ranks]
        for s in range(B):
            r_ = orc[s].step(streams[s][0][t], streams[s][1][t], streams[s][2][t], streams[s][3][t])
            ctx = (t, s)
            for r in range(W):
                experts, gates, _, summ = reads[r]
                assert experts[s].tolist() == r_["experts"], ctx
                sm = summ[s]
                assert (sm["hits"], sm["n_attended"], sm["fetch_elements"]) == (
                    r_["hits"], r_["n_attended"], r_["fetch_elements"]), ctx
                assert (sm["pages_before"], sm["pages_after"]) == (r_["pages_before"], r_["pages_after"])
                y = ys[r][s].double().cpu().numpy()
                assert rel_l2(y, r_["y"]) <= 2e-5, (ctx, r, rel_l2(y, r_["y"]))
            want = r_["evictions"]
            got_ow = sorted(tuple(e) for e in want if e[6] == 2)
            mine_ow = []
            for r in range(W):
                mine = [(e.step, e.entry_id, e.token_id, e.expert_id, e.device, e.score, REASON[e.reason])
                        for e in evs[r] if e.stream == s]
                mine_ow += [m for m in mine if m[6] == 2]
                sched_mine = [m for m in mine if m[6] != 2]
                assert sched_mine == [e for e in want if e[6] != 2 and e[4] == r], (ctx, r)
            assert sorted(mine_ow) == got_ow, ctx
            toks, exps = [], []
            for r in range(W):
                tk, ex, _ = ranks[r].read_attended(s)
                toks += list(tk)
                exps += list(ex)
            assert sorted(zip(toks, exps)) == list(zip(r_["att_token"], r_["att_expert"])), ctx
    for s in range(B):
        st = orc[s].slots()
        for r in range(W):
            a = ranks[r].slots(s)
            sl = slice(r * n_dev_slots, (r + 1) * n_dev_slots)
            assert np.array_equal(a["id"], st["id"][sl])
            live = a["id"] != 0
            for key in ("shard_seq", "token", "expert", "insert_step", "last_access", "freq"):
                assert np.array_equal(a[key][live], st[key][sl][live]), key
        for r in range(W):
            rs, ro = ranks[r].router_state(s), orc[s].router_state()
            assert np.array_equal(rs["miss"], ro["miss"]) and np.array_equal(rs["usage"], ro["usage"])
            assert ranks[r].scheduler_state(s)["step"] == orc[s].sched_state()["step"]
