# SPDX-License-Identifier: Apache-2.0
"""The reference's component-level known-answer tests, run through the GPU
component API (include/pikv_b200.h "component API";
paper_2508_06526_b200/components.py mirrors the reference classes):
test_kvstore.cpp:72-245, test_router.cpp:34-291, test_scheduler.cpp:75-317,
test_compressor.cpp:130-161 and test_pipeline.cpp:80-119 (attention on
stored entries).  Quoted numbers are the reference's."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle_bind import normal_vector  # noqa: E402
from paper_2508_06526_b200.components import (Codec, EntryMeta, KVEntry, KVStore,  # noqa: E402
                                              RouterState, adapt, record_miss, route, route_logits,
                                              score_entry)
from paper_2508_06526_b200.config import (CompressorConfig, ModelConfig, RouterConfig,  # noqa: E402
                                          SchedulerConfig, StoreConfig)
from paper_2508_06526_b200.engine import PikvError  # noqa: E402


def make_entry(token, expert, width, fill=1.0, **meta):
    return KVEntry(token_id=token, expert_id=expert, key=np.full(width, fill), value=np.full(width, fill),
                   meta=EntryMeta(**meta))


def small_model(d, S, G=1):  # test_kvstore.cpp:26-37
    return ModelConfig(d=d, head_width=1, E=8, k=1, S=S, G=G, rho=1.0)


# ------------------------------------------------------------ KVStore ----
def test_ring_fill_then_fifo_overwrite():  # test_kvstore.cpp:72-88 (one shard of capacity 4)
    st = KVStore(small_model(2, 4), StoreConfig(n_tok=1, n_exp=1))
    assert st.insert(make_entry(0, 0, 2)) is None
    assert st.live_count(0, 0) == 1
    for t in range(1, 4):
        st.insert(make_entry(t, 0, 2))
    assert st.live_count(0, 0) == 4
    fifth = st.insert(make_entry(4, 0, 2))
    assert fifth is not None and fifth.token_id == 0  # 5th insert displaces the 1st
    for t in range(5, 7):
        st.insert(make_entry(t, 0, 2))
    eighth = st.insert(make_entry(7, 0, 2))
    assert eighth is not None and eighth.token_id == 3
    assert st.live_count(0, 0) == 4


def test_ring_fifo_matches_tail_list():  # test_kvstore.cpp:90-107
    rng = np.random.default_rng(17)
    for trial in range(12):
        cap = int(rng.integers(1, 9))
        n = int(rng.integers(0, 40))
        st = KVStore(small_model(2, cap), StoreConfig(n_tok=1, n_exp=1))
        for t in range(n):
            st.insert(make_entry(t, 0, 2))
        got = sorted(e.token_id for _, _, e in st.for_each_live())
        assert got == list(range(max(0, n - cap), n))


def test_insert_width_checked():  # test_kvstore.cpp:109-112
    st = KVStore(small_model(4, 4), StoreConfig(n_tok=4, n_exp=4))
    with pytest.raises(PikvError) as ei:
        st.insert(make_entry(0, 0, 3))
    assert ei.value.kind == "InvalidEntry"


def test_retrieve_filters_by_expert_and_position():  # test_kvstore.cpp:114-160
    st = KVStore(small_model(4, 16), StoreConfig(n_tok=8, n_exp=8))
    r = st.retrieve([2], 100, 100)  # empty store misses
    assert r.entries == [] and r.missed_experts == [2] and st.stats().misses == 1
    st = KVStore(small_model(4, 16), StoreConfig(n_tok=8, n_exp=8))
    st.insert(make_entry(3, 2, 4))
    r = st.retrieve([2], 10, 10)
    assert len(r.entries) == 1 and r.entries[0].token_id == 3
    assert r.entries[0].meta.freq == 1 and r.entries[0].meta.last_access_step == 10
    assert r.missed_experts == []
    st = KVStore(small_model(4, 16), StoreConfig(n_tok=8, n_exp=8))
    alls = []
    for t in range(12):
        st.insert(make_entry(t, t % 3, 4))
        alls.append((t, t % 3))
    r = st.retrieve([0, 2], 12, 12)
    assert all(e.expert_id in (0, 2) for e in r.entries)
    assert [e.token_id for e in r.entries] == sorted(t for t, e in alls if e in (0, 2))
    older = st.retrieve([0, 2], 6, 12)
    assert all(e.token_id < 6 for e in older.entries)


def test_retrieval_completeness_before_overwrite():  # test_kvstore.cpp:162-176
    st = KVStore(small_model(4, 64), StoreConfig(n_tok=16, n_exp=8))
    rng = np.random.default_rng(5)
    n = 100
    for t in range(n):
        st.insert(make_entry(t, int(rng.integers(0, 8)), 4))
    assert st.stats().overwrites == 0
    r = st.retrieve(list(range(8)), n, n)
    assert len(r.entries) == n and len({e.token_id for e in r.entries}) == n


def test_memory_accounting():  # test_kvstore.cpp:178-205
    st = KVStore(small_model(32, 8), StoreConfig(n_tok=1, n_exp=1))
    assert st.memory_bytes() == 0
    m = small_model(32, 8)
    m.elem_bytes = 2
    st = KVStore(m, StoreConfig(n_tok=1, n_exp=1))
    assert st.shards_per_device() == 1
    for t in range(8):
        st.insert(make_entry(t, 0, 32))
    assert st.live_count(0, 0) == 8 and st.memory_bytes() == 1024
    m = small_model(16, 8)
    m.elem_bytes = 2
    st = KVStore(m, StoreConfig(n_tok=2, n_exp=1))
    for t in (0, 2, 4):
        st.insert(make_entry(t, 0, 16))
    for t in (1, 3, 5, 7, 9):
        st.insert(make_entry(t, 0, 16))
    assert st.live_count(0, 0) == 3 and st.live_count(0, 1) == 5
    assert st.memory_bytes() == 512


def test_bytes_live_bound():  # test_kvstore.cpp:207-218
    m = small_model(8, 4, 2)
    m.elem_bytes = 2
    st = KVStore(m, StoreConfig(n_tok=8, n_exp=8))
    bound = 2 * st.devices() * st.shards_per_device() * 8 * 4 * 2
    rng = np.random.default_rng(11)
    for t in range(120):
        st.insert(make_entry(t, int(rng.integers(0, 8)), 8))
        assert st.memory_bytes() <= bound


def test_erase_removes_a_live_entry():  # test_kvstore.cpp:220-230
    st = KVStore(small_model(4, 8), StoreConfig(n_tok=4, n_exp=4))
    st.insert(make_entry(0, 1, 4))
    st.insert(make_entry(1, 1, 4))
    r = st.retrieve([1], 10, 10)
    assert len(r.entries) == 2
    i = r.entries[0].id
    assert st.erase(i)
    assert not st.erase(i)
    assert st.live_entries() == 1


def test_snapshot_ordered_and_complete():  # test_kvstore.cpp:232-243
    st = KVStore(small_model(4, 8), StoreConfig(n_tok=4, n_exp=4))
    for t in range(6):
        st.insert(make_entry(t, t % 2, 4))
    snap = st.snapshot(6)
    assert len(snap) == 6
    keys = [(int(r["device"]), int(r["shard"]), int(r["token"])) for r in snap]
    assert keys == sorted(keys)


def test_insert_returns_displaced_payload_and_meta():
    """KVStore::insert returns the displaced entry by value (kvstore.hpp:106-108)."""
    st = KVStore(small_model(3, 2), StoreConfig(n_tok=1, n_exp=1), n_layers=2)
    st.insert(KVEntry(0, 0, np.array([1., 2., 3.]), np.array([4., 5., 6.]),
                      EntryMeta(7, 8, 9, 0.25, [0.5, 1.5])))
    st.insert(make_entry(1, 0, 3))
    d = st.insert(make_entry(2, 0, 3))
    assert d.token_id == 0 and d.id == 1 and d.shard_seq == 0
    assert list(d.key) == [1, 2, 3] and list(d.value) == [4, 5, 6]
    assert (d.meta.insert_step, d.meta.last_access_step, d.meta.freq) == (7, 8, 9)
    assert d.meta.attn_mass == 0.25 and d.meta.per_layer_scores == [0.5, 1.5]


# ------------------------------------------------------------- router ----
def rc(strategy, k, **kw):
    return RouterConfig(strategy=strategy, k=k, **kw)


def test_base_round_robin():  # test_router.cpp:34-44
    st = RouterState.init(4, 8, 1)
    for t in range(4):
        d = route(np.zeros(8), st, rc("Base", 1))
        assert d.experts == [t] and abs(d.gates[0] - 1.0) < 1e-12


def test_topk_gates():  # test_router.cpp:46-54
    d = route_logits([2, 1, 0, -1], RouterState.init(4, 4, 1), rc("TopK", 2))
    assert d.experts == [0, 1]
    assert abs(d.gates[0] - 0.7310585786300049) <= 1e-12
    assert abs(d.gates[1] - 0.2689414213699951) <= 1e-12


def test_load_balanced_penalty():  # test_router.cpp:56-63
    st = RouterState.init(4, 4, 1)
    st._engine(rc("LoadBalanced", 1, alpha=0.5))
    st.set(load=[10, 0, 0, 0])
    assert route_logits([1, 1, 1, 1], st, rc("LoadBalanced", 1, alpha=0.5)).experts[0] == 1


def test_cache_aware_zero_misses():  # test_router.cpp:65-75
    a = route_logits([0.3, 0.1, 0.9, 0.2], RouterState.init(4, 4, 1), rc("TopK", 2))
    b = route_logits([0.3, 0.1, 0.9, 0.2], RouterState.init(4, 4, 1), rc("CacheAware", 2, lambda_miss=3.0))
    assert a.experts == b.experts and abs(a.gates[0] - b.gates[0]) < 1e-12


def test_record_miss():  # test_router.cpp:77-86
    st = RouterState.init(4, 4, 1)
    record_miss(st, 2)
    assert list(st.miss_counts) == [0, 0, 1, 0]
    record_miss(st, 2)
    assert st.miss_counts[2] == 2
    for bad in (4, -1):
        with pytest.raises(PikvError) as ei:
            record_miss(st, bad)
        assert ei.value.kind == "InvalidArgument"


def test_adapt_bandit_rule():  # test_router.cpp:88-117
    from paper_2508_06526_b200.components import RoutingDecision
    cfg = rc("Adaptive", 2, bandit_step=0.1)
    d = RoutingDecision([0, 2], [], [])
    st = RouterState.init(4, 4, 1)
    st._engine(cfg)
    st.set(bias=[0.5] * 4)
    adapt(st, d, 0.5, cfg)
    assert np.allclose(st.bandit_bias, 0.5)
    st = RouterState.init(4, 4, 1)
    adapt(st, d, 1.0, cfg)
    assert np.allclose(st.bandit_bias, [0.1, 0.0, 0.1, 0.0])
    for bad in (1.5, -0.1):
        with pytest.raises(PikvError):
            adapt(st, d, bad, cfg)
    cap = rc("Adaptive", 2, bandit_step=10.0)
    for _ in range(50):
        adapt(st, d, 1.0, cap)
    assert st.bandit_bias[0] <= cap.bias_cap


def test_adaptive_bandit_learns():  # test_router.cpp:119-135
    st = RouterState.init(8, 16, 42)
    cfg = rc("Adaptive", 2, bandit_step=0.05)
    qs = normal_vector(42, 1000 * 16).reshape(1000, 16)  # Rng(42).normal_vector(16) x 1000
    for t in range(1000):
        d = route(qs[t], st, cfg)
        adapt(st, d, 1.0 if 0 in d.experts else 0.0, cfg)
    assert int(np.argmax(st.bandit_bias)) == 0


@pytest.mark.parametrize("strategy", ["TopK", "LoadBalanced", "CacheAware", "EntropyLB", "Adaptive",
                                      "Hierarchical"])
def test_sparsity_k_distinct(strategy):  # test_router.cpp:136-161
    rng = np.random.default_rng(19)
    st = RouterState.init(16, 8, 7)
    for k in (1, 2, 4):
        cfg = rc(strategy, k, groups=4 if strategy == "Hierarchical" else 1)
        for _ in range(10):
            d = route(rng.standard_normal(8), st, cfg)
            assert len(d.experts) == k and len(set(d.experts)) == k
            assert abs(sum(d.gates) - 1.0) < 1e-12


def test_topk_shift_invariance():  # test_router.cpp:163-196
    rng = np.random.default_rng(3)
    for _ in range(20):
        lg = rng.standard_normal(8)
        a = route_logits(lg, RouterState.init(8, 4, 1), rc("TopK", 3))
        b = route_logits(lg + 5.0, RouterState.init(8, 4, 1), rc("TopK", 3))
        assert a.experts == b.experts and np.allclose(a.gates, b.gates, rtol=1e-12)


def test_hierarchical_groups_one_is_topk():  # test_router.cpp:248-264
    rng = np.random.default_rng(23)
    for _ in range(20):
        lg = rng.standard_normal(8)
        a = route_logits(lg, RouterState.init(8, 4, 1), rc("TopK", 2))
        b = route_logits(lg, RouterState.init(8, 4, 1), rc("Hierarchical", 2, groups=1))
        assert a.experts == b.experts


def test_hierarchical_ragged_clusters():  # test_router.cpp:266-279
    d = route_logits([0.0, 0.1, 0.2, 5.0, 4.0], RouterState.init(5, 4, 1), rc("Hierarchical", 2, groups=2))
    assert sorted(d.experts) == [3, 4]


def test_nan_is_numerical_error():  # test_router.cpp:281-291
    st = RouterState.init(4, 4, 1)
    with pytest.raises(PikvError) as ei:
        route_logits([0.0, float("nan"), 1.0, 2.0], st, rc("TopK", 2))
    assert ei.value.kind == "NumericalError"
    assert route_logits([0.0, 1.0, 3.0, 2.0], st, rc("TopK", 2)).experts == [2, 3]  # state unharmed


# ---------------------------------------------------------- scheduler ----
def meta_entry(attn, ins, la, freq, token=100, layers=()):
    return KVEntry(token_id=token, key=np.array([1.0, 0.0]), value=np.array([0.5, 0.5]),
                   meta=EntryMeta(ins, la, freq, attn, list(layers)))


def test_score_table_strategies():  # test_scheduler.cpp:75-154
    def sc(e, strat, now=5, **kw):
        return score_entry(e, SchedulerConfig(strategy=strat, **kw), now)
    assert sc(meta_entry(0.37, 0, 0, 0), "H2O") == pytest.approx(0.37)
    assert sc(meta_entry(0, 0, 3, 0), "LRU") == pytest.approx(-2.0)
    assert sc(meta_entry(0, 0, 3, 3), "LRUPlus", lambda_freq=0.5) == pytest.approx(-0.5)
    assert sc(meta_entry(0.2, 5, 5, 4), "AdaKV", adakv_weights=[1.0, 0.5]) == pytest.approx(2.2)
    sl = dict(tau=10, sink=4)
    young = sc(meta_entry(0, 95, 95, 0, 100), "SL", 100, **sl)
    assert young == pytest.approx(1.0)
    assert sc(meta_entry(0, 0, 0, 0, 100), "SL", 100, **sl) == pytest.approx(0.0)
    assert sc(meta_entry(0, 0, 0, 0, 2), "SL", 100, **sl) > young
    fx = dict(flex_plan=[1.0, 0.5, 0.0], flex_bucket=10)
    assert sc(meta_entry(0, 100, 100, 0), "Flex", 100, **fx) == 1.0
    assert sc(meta_entry(0, 85, 85, 0), "Flex", 100, **fx) == 0.5
    assert sc(meta_entry(0, 0, 0, 0), "Flex", 100, **fx) == 0.0
    rng = np.random.default_rng(3)
    for _ in range(30):  # duo sums the per-layer scores exactly (sequentially)
        layers = list(rng.random(int(rng.integers(1, 7))))
        want = 0.0
        for a in layers:
            want += a
        assert sc(meta_entry(0, 0, 0, 0, layers=layers), "Duo") == want
    assert sc(meta_entry(0, 0, 0, 0), "Duo") == 0.0  # empty per_layer_scores
    with pytest.raises(PikvError) as ei:
        sc(meta_entry(0, 0, 0, 0), "QUEST")
    assert ei.value.kind == "NotFitted"


class StoreFixture:  # test_scheduler.cpp:38-70
    def __init__(self, capacity, page_size, d=2):
        m = ModelConfig(d=d, head_width=1, E=4, k=1, S=capacity, G=1)
        self.store = KVStore(m, StoreConfig(n_tok=1, n_exp=1), page_size=page_size)
        self.d = d

    def insert(self, attn, token):
        self.store.insert(KVEntry(token_id=token, expert_id=0, key=np.ones(self.d), value=np.ones(self.d),
                                  meta=EntryMeta(attn_mass=attn)))


def test_evict_page_budget_live_store():  # test_scheduler.cpp:236-259
    fx = StoreFixture(16, 1)
    cfg = SchedulerConfig(strategy="H2O", page_size=1, budget_pages=2)
    for a, t in ((5.0, 0), (1.0, 1), (3.0, 2), (2.0, 3)):
        fx.insert(a, t)
    rep = fx.store.evict(cfg, 4)
    assert (rep.pages_before, rep.pages_after) == (4, 2)
    assert [e.token_id for e in rep.evicted] == [1, 3]
    assert fx.store.live_entries() == 2
    assert fx.store.evict(cfg, 5).evicted == []


def test_evict_pages_group_page_size():  # test_scheduler.cpp:261-275
    fx = StoreFixture(64, 4)
    cfg = SchedulerConfig(strategy="H2O", page_size=4, budget_pages=3)
    rng = np.random.default_rng(17)
    for t in range(40):
        fx.insert(float(rng.random()), t)
    rep = fx.store.evict(cfg, 40)
    assert (rep.pages_before, rep.pages_after) == (10, 3)
    assert fx.store.live_entries() == 12 and len(rep.evicted) == 28


def test_evict_after_erase_holes():
    """Pages with holes left by KVStore::erase still aggregate / evict their
    remaining members only (the reference groups live entries by page)."""
    fx = StoreFixture(64, 4)
    cfg = SchedulerConfig(strategy="LRU", page_size=4, budget_pages=2)
    for t in range(16):
        fx.insert(0.0, t)
    ids = {e.token_id: e.id for _, _, e in fx.store.for_each_live()}
    for t in (0, 5, 6, 9):  # page 0 loses its first, page 1 its middle members
        assert fx.store.erase(ids[t])
    rep = fx.store.evict(cfg, 20)
    assert (rep.pages_before, rep.pages_after) == (4, 2)
    # LRU at now 20, all last accessed at 0: aggregates -60 / -40 / -60 / -80
    # -> page 3, then page 0 (tie with page 2 broken by the oldest id)
    assert [e.token_id for e in rep.evicted] == [12, 13, 14, 15, 1, 2, 3]
    assert all(e.score == -20.0 for e in rep.evicted)
    assert sorted(e.token_id for _, _, e in fx.store.for_each_live()) == [4, 7, 8, 10, 11]


def test_adakv_threshold_rule():  # test_scheduler.cpp:277-317
    cfg = SchedulerConfig(strategy="AdaKV", adakv_step=0.1, target_hit=0.9, theta0=0.5, hit_decay=0.0)
    fx = StoreFixture(4, 16)
    fx.store.set_scheduler_state(theta=0.5, running_hit=0.0)
    fx.store.observe_hits(cfg, 7, 10)
    fx.store.adakv_update(cfg)
    assert fx.store.scheduler_state()["theta"] == pytest.approx(0.52)
    fx.store.set_scheduler_state(theta=0.5, running_hit=0.0)
    fx.store.observe_hits(cfg, 9, 10)
    fx.store.adakv_update(cfg)
    assert fx.store.scheduler_state()["theta"] == pytest.approx(0.5)
    fx.store.set_scheduler_state(theta=0.5, running_hit=0.0)
    fx.store.observe_hits(cfg, 1, 10)
    prev = 0.5
    for _ in range(50):
        fx.store.adakv_update(cfg)
        th = fx.store.scheduler_state()["theta"]
        assert th > prev
        prev = th


# ---------------------------------------------------- attention, codec ----
def test_attention_on_stored_entries():  # test_pipeline.cpp:80-119
    st = KVStore(small_model(2, 8), StoreConfig(n_tok=1, n_exp=1))
    y, w = st.attention([1.0, 0.0], [])
    assert list(y) == [0.0, 0.0] and len(w) == 0
    st.insert(KVEntry(0, 0, np.array([1.0, 0.0]), np.array([3.0, 4.0])))
    y, w = st.attention([1.0, 0.0], [0])
    assert np.allclose(y, [3, 4]) and np.allclose(w, [1.0])
    st.insert(KVEntry(1, 0, np.array([1.0, 0.0]), np.array([5.0, 6.0])))
    y, w = st.attention([1.0, 0.0], [0, 1])  # identical keys: 0.5 / 0.5
    assert np.allclose(w, [0.5, 0.5]) and np.allclose(y, [4, 5])


def test_fastv_crop_and_zero_fill():  # test_compressor.cpp:130-142
    c = Codec.fit("FastV", [[0.0, 0.0], [1.0, 1.0]], CompressorConfig(rank=1))
    assert list(c.encode_vector([3, 4])) == [3]
    assert list(c.decode_vector(c.encode_vector([3, 4]))) == [3, 0]
    assert c.reconstruction_error([3, 4]) == pytest.approx(0.8, rel=1e-6)


def test_prune_keeps_high_variance():  # test_compressor.cpp:144-161
    c = Codec.fit("Prune", [[1, 7], [-3, 7], [2, 7], [-1, 7]], CompressorConfig(rank=1), prune_frac=0.5)
    assert c.zero_set() == [1]
    assert list(c.encode_vector([3, 4])) == [3]
    assert list(c.decode_vector(c.encode_vector([3, 4]))) == [3, 0]
    eps = c.reconstruction_error([3, 4])
    assert eps * eps * (9.0 + 16.0) == pytest.approx(16.0, rel=1e-6)


def test_lowrank_codec_matches_projection():  # compressor.cpp:318-340
    rng = np.random.default_rng(4)
    d, r = 16, 4
    basis = np.linalg.qr(rng.standard_normal((d, d)))[0][:, :r].T.astype(np.float32)  # [r][d]
    c = Codec("LowRank", d, r, basis=basis[None])
    x = rng.standard_normal(d)
    y = c.encode_vector(x)
    assert np.allclose(y, basis @ x, rtol=1e-5, atol=1e-5)
    assert np.allclose(c.decode_vector(y), basis.T @ (basis @ x), rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("E,k,d", [(16, 2, 4096), (64, 4, 1024)])
def test_fast_routing_flip_rate(E, k, d):
    """PIKV_ROUTE_FAST (tree-reduced fp64 logits) against the exact sequential
    chain (router.cpp:224-229) on the same 4000 N(0,1) queries: logits agree
    to rounding order (<= 1e-12 relative to the row norm), and the selected
    experts flip only on near-ties (the rate is reported; bound 1e-3)."""
    rng = np.random.default_rng(E)
    ex, fa = RouterState(E, d, 7), RouterState(E, d, 7, route_mode="fast")
    cfg = rc("TopK", k)
    flips, worst = 0, 0.0
    n = 4000
    for q in rng.standard_normal((n, d)):
        a, b = route(q, ex, cfg), route(q, fa, cfg)
        la, lb = np.array(a.logits), np.array(b.logits)
        worst = max(worst, float(np.max(np.abs(la - lb)) / max(np.linalg.norm(la), 1e-300)))
        flips += a.experts != b.experts
    print("fast routing E%d k%d d%d: %d / %d selections differ, logit rel diff %.2e" % (E, k, d, flips, n, worst))
    assert worst <= 1e-12
    assert flips / n <= 1e-3
