# SPDX-License-Identifier: Apache-2.0
"""The reference's component API over the GPU engine (include/pikv_b200.h,
"component API"): ``KVStore`` (kvstore.hpp:100-159), ``RouterState`` with
``route`` / ``route_logits`` / ``record_miss`` / ``adapt`` (router.hpp:41-79),
``SchedulerState`` with ``score_entry`` / ``evict`` / ``observe_hits`` /
``adakv_update`` (scheduler.hpp:49-129), ``attention`` over stored entries
(pipeline.hpp:46-47) and ``Codec`` (compressor.hpp:57-80).

Every call is a CUDA kernel on the engine's HBM state of one stream; these
classes only marshal arguments.  Differences from the reference, each forced
by a device-resident store: the store is created with the scheduler's page
size (its page records are maintained on insert), a RouterState is sized
for one k at a time (re-sized transparently, state carried over), and
retrieved entries are host copies (RetrievalResult holds values, not
pointers into the store).
"""
from __future__ import annotations

import ctypes
import dataclasses
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from ._capi import PikvEntry, PikvEvictRecord, check, lib
from .config import (CompressorConfig, EngineConfig, ModelConfig, RouterConfig, SchedulerConfig,
                     StoreConfig, REASON)
from .engine import Engine, ShardId, shard_assign

ROUTER_SALT = 0x2545F4914F6CDD1D  # pipeline.cpp:16 (the engine seeds W_r with seed ^ salt)


def _p(a):
    return None if a is None else a.ctypes.data


# ------------------------------------------------------------------ types --
@dataclass
class EntryMeta:  # types.hpp:11-24
    insert_step: int = 0
    last_access_step: int = 0
    freq: int = 0
    attn_mass: float = 0.0
    per_layer_scores: List[float] = field(default_factory=list)


@dataclass
class KVEntry:  # types.hpp:27-34
    token_id: int = 0
    expert_id: int = 0
    key: np.ndarray = field(default_factory=lambda: np.zeros(0))
    value: np.ndarray = field(default_factory=lambda: np.zeros(0))
    meta: EntryMeta = field(default_factory=EntryMeta)
    id: int = 0
    shard_seq: int = 0


@dataclass
class RetrievalResult:  # kvstore.hpp:81-87 (entries are host copies here)
    entries: List[KVEntry]
    missed_experts: List[int]
    slots: np.ndarray


@dataclass
class StoreStats:  # kvstore.hpp:74-79
    inserts: int = 0
    overwrites: int = 0
    retrievals: int = 0
    misses: int = 0


@dataclass
class RoutingDecision:  # router.hpp:58-62
    experts: List[int]
    gates: List[float]
    logits: List[float]


@dataclass
class EvictionRecord:  # scheduler.hpp:90-98
    step: int
    entry_id: int
    token_id: int
    expert_id: int
    device: int
    score: float
    reason: str


@dataclass
class EvictionReport:  # scheduler.hpp:100-104
    evicted: List[EvictionRecord]
    pages_before: int
    pages_after: int


def _entry_c(e: KVEntry, has_layers: bool) -> PikvEntry:
    c = PikvEntry()
    c.token_id, c.expert_id = int(e.token_id), int(e.expert_id)
    c.has_layers = int(has_layers)
    c.insert_step, c.last_access_step = int(e.meta.insert_step), int(e.meta.last_access_step)
    c.freq, c.attn_mass = int(e.meta.freq), float(e.meta.attn_mass)
    return c


def _entry_py(c: PikvEntry, key, value, layers) -> KVEntry:
    return KVEntry(token_id=c.token_id, expert_id=c.expert_id, key=key, value=value, id=c.id,
                   shard_seq=c.shard_seq,
                   meta=EntryMeta(c.insert_step, c.last_access_step, c.freq, c.attn_mass,
                                  list(layers) if c.has_layers else []))


# ---------------------------------------------------------------- KVStore --
class KVStore:
    """Expert-sharded store (kvstore.hpp:100-159) held in HBM by a one-stream
    engine.  ``kv_dtype`` / ``codec`` select the stored format (fp32 keeps the
    reference's values exactly for fp32-representable inputs)."""

    def __init__(self, model: ModelConfig, store: StoreConfig, *, page_size: int = 16,
                 n_heads: int = 1, n_layers: int = 0, kv_dtype: str = "f32", codec: str = "Identity",
                 pool_entries: int = 0, sched: Optional[SchedulerConfig] = None, device: int = 0):
        cfg = EngineConfig()
        dp = model.d_prime()  # the store holds d'-wide (compressed) vectors
        cfg.model = dataclasses.replace(model, d=dp, rho=1.0, head_width=min(model.head_width, dp))
        cfg.store = store
        cfg.router = RouterConfig(strategy="TopK", k=1)
        cfg.scheduler = dataclasses.replace(sched or SchedulerConfig(), page_size=page_size)
        cfg.compressor = CompressorConfig(scheme=codec)
        cfg.n_heads, cfg.n_layers, cfg.kv_dtype, cfg.batch = n_heads, n_layers, kv_dtype, 1
        cfg.pool_entries = pool_entries
        self.cfg = cfg
        self.engine = Engine(cfg, device=device)
        self.h = self.engine.h
        self.d_prime = cfg.model.d
        self.page_size = page_size
        self.n_layers = n_layers

    # kvstore.hpp:105
    def locate(self, token_id: int, expert_id: int) -> ShardId:
        s = self.cfg.store
        return shard_assign(int(token_id), int(expert_id), s.n_tok, s.n_exp, self.cfg.model.G, s.additive)

    def insert(self, entry: KVEntry) -> Optional[KVEntry]:
        """KVStore::insert (kvstore.cpp:107-120); returns the displaced entry."""
        from .engine import PikvError
        k = np.ascontiguousarray(entry.key, dtype=np.float32).ravel()
        v = np.ascontiguousarray(entry.value, dtype=np.float32).ravel()
        if k.size != self.d_prime or v.size != self.d_prime:  # kvstore.cpp:108-111
            raise PikvError(3, "KVStore::insert: entry width != d'")
        pl = entry.meta.per_layer_scores
        has = len(pl) > 0 and self.n_layers > 0
        layers = np.zeros(max(self.n_layers, 1))
        layers[:min(len(pl), self.n_layers)] = pl[:self.n_layers]
        ec = _entry_c(entry, has)
        dsp = PikvEntry()
        dk = np.zeros(self.d_prime, dtype=np.float32)
        dv = np.zeros(self.d_prime, dtype=np.float32)
        dl = np.zeros(max(self.n_layers, 1))
        flag = ctypes.c_int32(0)
        check(lib().pikv_store_insert_host(self.h, 0, 1, ctypes.addressof(ec), _p(k), _p(v),
                                           _p(layers) if has else None, ctypes.addressof(dsp),
                                           _p(dk), _p(dv), _p(dl), ctypes.addressof(flag)))
        if not flag.value:
            return None
        return _entry_py(dsp, dk, dv, dl[:self.n_layers])

    def retrieve(self, experts: Sequence[int], since: int, now: int) -> RetrievalResult:
        ex = np.ascontiguousarray(experts, dtype=np.int32)
        n, nm = ctypes.c_int32(0), ctypes.c_int32(0)
        cap = self.slot_count()
        slots = np.zeros(cap, dtype=np.int64)
        missed = np.zeros(max(len(ex), 1), dtype=np.int32)
        check(lib().pikv_store_retrieve_host(self.h, 0, _p(ex), len(ex), int(since), int(now),
                                             _p(slots), cap, ctypes.byref(n), _p(missed),
                                             ctypes.byref(nm)))
        slots = slots[:n.value]
        return RetrievalResult(self.entries_at(slots), [int(x) for x in missed[:nm.value]], slots)

    def entries_at(self, slots) -> List[KVEntry]:
        """Host copies of the entries in the given stream-local slots."""
        slots = np.ascontiguousarray(slots, dtype=np.int64)
        if len(slots) == 0:
            return []
        st = self.engine.slots(0)
        k, v = self.engine.read_entries(0, slots)
        nl = self.n_layers
        out = []
        for i, s in enumerate(slots):
            layers = list(st["per_layer"][s * nl:(s + 1) * nl]) if nl else []
            out.append(KVEntry(token_id=int(st["token"][s]), expert_id=int(st["expert"][s]),
                               key=k[i], value=v[i], id=int(st["id"][s]),
                               shard_seq=int(st["shard_seq"][s]),
                               meta=EntryMeta(int(st["insert_step"][s]), int(st["last_access"][s]),
                                              int(st["freq"][s]), float(st["attn_mass"][s]), layers)))
        return out

    def erase(self, entry_id: int) -> bool:
        ok = ctypes.c_int32(0)
        check(lib().pikv_store_erase_host(self.h, 0, int(entry_id), ctypes.byref(ok)))
        return bool(ok.value)

    def memory_bytes(self) -> int:
        return self.engine.store_stats(0)["memory_bytes"]

    def live_entries(self) -> int:
        return self.engine.store_stats(0)["live"]

    def stats(self) -> StoreStats:
        st = self.engine.store_stats(0)
        r, m = ctypes.c_uint64(0), ctypes.c_uint64(0)
        check(lib().pikv_store_counters_host(self.h, 0, ctypes.byref(r), ctypes.byref(m)))
        return StoreStats(st["inserts"], st["overwrites"], r.value, m.value)

    def devices(self) -> int:
        return self.cfg.model.G

    def shards_per_device(self) -> int:
        return self.slot_count() // (self.cfg.model.S * self.cfg.model.G)

    def slot_count(self) -> int:
        return int(lib().pikv_slot_count(self.h))

    def live_count(self, device: int, shard: int) -> int:
        """ShardBuffer::live_count of buffer(device, shard) (kvstore.hpp:41)."""
        live = np.zeros(self.devices() * self.shards_per_device(), dtype=np.int32)
        check(lib().pikv_ring_live_host(self.h, 0, _p(live)))
        return int(live[device * self.shards_per_device() + shard])

    def for_each_live(self):
        """(device, shard, KVEntry) of every live entry, device-major, slot order."""
        st = self.engine.slots(0)
        live = np.flatnonzero(st["id"] != 0)
        spd, S = self.shards_per_device(), self.cfg.model.S
        return [(int(s // S) // spd, int(s // S) % spd, e) for s, e in zip(live, self.entries_at(live))]

    def snapshot(self, now: int):
        return self.engine.snapshot(0, now)

    def attention(self, query, slots):
        """attention(q, entries) (pipeline.cpp:59-85) over stored entries, per
        head; returns (output [d'], weights [n] = mean over heads)."""
        q = np.ascontiguousarray(query, dtype=np.float32).ravel()
        sl = np.ascontiguousarray(slots, dtype=np.int64)
        y = np.zeros(self.d_prime, dtype=np.float32)
        a = np.zeros(max(len(sl), 1), dtype=np.float32)
        check(lib().pikv_attend_host(self.h, 0, _p(q), _p(sl), len(sl), _p(y), _p(a)))
        return y, a[:len(sl)]

    # -- scheduler on this store (scheduler.hpp:83-129) --------------------
    def _set_sched(self, cfg: SchedulerConfig):
        from .engine import PikvError
        if cfg.page_size != self.page_size:
            raise PikvError(2, "evict: the store was built for page_size %d" % self.page_size)
        c = dataclasses.replace(self.cfg, scheduler=cfg)
        check(lib().pikv_update_config(self.h, ctypes.byref(c.to_c())))
        self.cfg = c

    def evict(self, cfg: SchedulerConfig, now: int) -> EvictionReport:
        """evict(store, state, cfg, nullptr, now) (scheduler.cpp:262-330) with
        this store's SchedulerState."""
        self._set_sched(cfg)
        cap = self.slot_count()
        recs = (PikvEvictRecord * max(cap, 1))()
        n, pb, pa = ctypes.c_int32(0), ctypes.c_int32(0), ctypes.c_int32(0)
        check(lib().pikv_evict_host(self.h, 0, int(now), ctypes.addressof(recs), cap, ctypes.byref(n),
                                    ctypes.byref(pb), ctypes.byref(pa)))
        ev = [EvictionRecord(r.step, r.entry_id, r.token_id, r.expert_id, r.device, r.score,
                             REASON[r.reason]) for r in recs[:n.value]]
        return EvictionReport(ev, pb.value, pa.value)

    def scheduler_state(self):
        return self.engine.scheduler_state(0)

    def observe_hits(self, cfg: SchedulerConfig, hits: int, lookups: int):
        self._set_sched(cfg)
        check(lib().pikv_observe_hits(self.h, 0, int(hits), int(lookups)))

    def adakv_update(self, cfg: SchedulerConfig):
        self._set_sched(cfg)
        check(lib().pikv_adakv_update(self.h, 0))

    def set_scheduler_state(self, theta=None, running_hit=None, step=None):
        t = None if theta is None else ctypes.c_double(theta)
        r = None if running_hit is None else ctypes.c_double(running_hit)
        s = None if step is None else ctypes.c_uint64(step)
        check(lib().pikv_write_sched_state_host(self.h, 0, *(None if x is None else ctypes.addressof(x)
                                                             for x in (t, r, s))))


def score_entry(entry: KVEntry, cfg: SchedulerConfig, now: int, n_layers: int = 0) -> float:
    """score_entry (scheduler.cpp:181-229) of one entry's metadata, on the GPU."""
    return float(score_entries([entry], cfg, now, n_layers)[0])


def score_entries(entries: Sequence[KVEntry], cfg: SchedulerConfig, now: int, n_layers: int = 0):
    ec = EngineConfig()
    ec.scheduler = cfg
    nl = max([n_layers] + [len(e.meta.per_layer_scores) for e in entries])
    ec.n_layers = nl
    arr = (PikvEntry * max(len(entries), 1))()
    layers = np.zeros((max(len(entries), 1), max(nl, 1)))
    for i, e in enumerate(entries):
        pl = e.meta.per_layer_scores
        arr[i] = _entry_c(e, len(pl) > 0)
        layers[i, :len(pl)] = pl
    out = np.zeros(max(len(entries), 1))
    check(lib().pikv_score_entries_host(ctypes.byref(ec.to_c()), ctypes.addressof(arr),
                                        _p(layers) if nl else None, len(entries), int(now), _p(out)))
    return out[:len(entries)]


# ------------------------------------------------------------ RouterState --
class RouterState:
    """RouterState::init(experts, width, seed) (router.cpp:54-67) on the GPU:
    W_r = Rng(seed) N(0, 1/d); load / usage / miss / bandit bias in HBM."""

    def __init__(self, experts: int, width: int, seed: int, device: int = 0, route_mode: str = "exact"):
        self.experts, self.width, self.seed, self.device = experts, width, seed, device
        self.route_mode = route_mode  # "fast": tree-reduced fp64 logits (PIKV_ROUTE_FAST)
        self._eng = None
        self._k = None
        self._cfg = None

    @classmethod
    def init(cls, experts: int, width: int, seed: int):
        return cls(experts, width, seed)

    def _engine(self, rcfg: RouterConfig) -> Engine:
        if self._eng is not None and rcfg.k == self._k:
            if rcfg != self._cfg:
                c = dataclasses.replace(self._ecfg, router=rcfg)
                check(lib().pikv_update_config(self._eng.h, ctypes.byref(c.to_c())))
                self._ecfg, self._cfg = c, rcfg
            return self._eng
        carried = self.view() if self._eng is not None else None
        c = EngineConfig()
        c.model = ModelConfig(d=self.width, head_width=1, E=self.experts, k=rcfg.k, G=1, S=1)
        c.store = StoreConfig(n_tok=1, n_exp=1)
        c.router = rcfg
        c.unbounded_budget = True
        c.seed = self.seed ^ ROUTER_SALT  # W_r = Rng(cfg.seed ^ salt) = Rng(seed)
        c.route_mode = self.route_mode
        c.batch, c.n_layers, c.pool_entries = 1, 0, 16
        if self._eng is not None:
            self._eng.close()
        self._eng, self._k, self._cfg, self._ecfg = Engine(c, device=self.device), rcfg.k, rcfg, c
        if carried is not None:
            self.set(**carried)
        return self._eng

    def view(self):
        if self._eng is None:
            z = np.zeros(self.experts)
            return {"load": z, "usage": z.astype(np.uint64), "miss": z.astype(np.uint64),
                    "bias": z.copy(), "step": 0, "total_usage": 0}
        return self._eng.router_state(0)

    @property
    def load(self):
        return self.view()["load"]

    @property
    def miss_counts(self):
        return self.view()["miss"]

    @property
    def usage_counts(self):
        return self.view()["usage"]

    @property
    def bandit_bias(self):
        return self.view()["bias"]

    def set(self, load=None, usage=None, miss=None, bias=None, step=None, total_usage=None):
        eng = self._engine(self._cfg or RouterConfig())
        arr = [None if a is None else np.ascontiguousarray(a, dtype=dt)
               for a, dt in ((load, np.float64), (usage, np.uint64), (miss, np.uint64), (bias, np.float64))]
        st = None if step is None else ctypes.c_uint64(step)
        tu = None if total_usage is None else ctypes.c_uint64(total_usage)
        check(lib().pikv_write_router_state_host(eng.h, 0, *[_p(a) for a in arr],
                                                 None if st is None else ctypes.addressof(st),
                                                 None if tu is None else ctypes.addressof(tu)))


def _decision(eng, fn, *args) -> RoutingDecision:
    k, E = eng.k, eng.E
    ex = np.zeros(k, dtype=np.int32)
    g = np.zeros(k)
    lg = np.zeros(E)
    check(fn(eng.h, 0, *args, _p(ex), _p(g), _p(lg)))
    return RoutingDecision([int(x) for x in ex], list(g), list(lg))


def route(query, state: RouterState, cfg: RouterConfig) -> RoutingDecision:
    """route (router.cpp:216-234): exact fp64 logits, penalty, selection."""
    eng = state._engine(cfg)
    q = None if query is None else np.ascontiguousarray(query, dtype=np.float64)
    if q is not None and cfg.strategy != "Base" and q.size != state.width:
        from .engine import PikvError
        raise PikvError(1, "route: query width != d")
    return _decision(eng, lib().pikv_route_host, _p(q))


def route_logits(logits, state: RouterState, cfg: RouterConfig) -> RoutingDecision:
    eng = state._engine(cfg)
    lg = np.ascontiguousarray(logits, dtype=np.float64)
    if lg.size != state.experts:
        from .engine import PikvError
        raise PikvError(1, "route_logits: logit width != E")
    return _decision(eng, lib().pikv_route_logits_host, _p(lg))


def record_miss(state: RouterState, expert: int):
    eng = state._engine(state._cfg or RouterConfig())
    check(lib().pikv_record_miss(eng.h, 0, int(expert)))


def adapt(state: RouterState, decision: RoutingDecision, reward: float, cfg: RouterConfig):
    eng = state._engine(cfg if state._cfg is None or cfg.k == state._k else state._cfg)
    if cfg != state._cfg and cfg.k == state._k:
        eng = state._engine(cfg)
    ex = np.ascontiguousarray(decision.experts, dtype=np.int32)
    check(lib().pikv_router_adapt(eng.h, 0, _p(ex), len(ex), float(reward)))


# ------------------------------------------------------------------ Codec --
CODEC_ID = {"Identity": 0, "SVD": 1, "LoRA": 1, "LowRank": 1, "LoRAPlus": 2, "FastV": 3, "Prune": 4}


class Codec:
    """Codec (compressor.hpp:57-80) with encode_vector / decode_vector on the
    GPU.  Projection schemes take their basis (fitting is offline,
    PAPER.md:499); FastV and Prune fit here (Prune's column variances on the
    GPU, compressor.cpp:250-262)."""

    def __init__(self, scheme: str, d: int, r: int, basis=None, bias=None, kept=None, heads: int = 1):
        self.scheme, self.d, self.r, self.heads = scheme, d, r, heads
        self.basis = None if basis is None else np.ascontiguousarray(basis, dtype=np.float32)
        self.bias = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
        self.kept = None if kept is None else np.ascontiguousarray(kept, dtype=np.int32)

    @classmethod
    def fit(cls, scheme: str, calibration, cfg: CompressorConfig, prune_frac: float = 0.5):
        X = np.ascontiguousarray(calibration, dtype=np.float64)
        n, d = X.shape
        if scheme == "Identity":
            return cls(scheme, d, d)
        if scheme == "FastV":
            return cls(scheme, d, cfg.rank)
        if scheme == "Prune":
            var = np.zeros(d)
            check(lib().pikv_column_variance_host(_p(X), n, d, _p(var)))
            drop = int(np.ceil(prune_frac * d))
            keep = max(1, d - drop)
            order = sorted(range(d), key=lambda i: (-var[i], i))
            kept = np.sort(np.array(order[:keep], dtype=np.int32))
            return cls(scheme, d, keep, kept=kept[None])
        raise ValueError("fit: %s needs a basis (Codec(scheme, d, r, basis=...))" % scheme)

    def stored_width(self) -> int:
        return self.d if self.scheme == "Identity" else self.r * self.heads

    def zero_set(self):
        if self.scheme != "Prune":
            return []
        return sorted(set(range(self.d)) - set(int(x) for x in self.kept.ravel()))

    def _call(self, fn, x, w_in, w_out):
        x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1, w_in)
        y = np.zeros((x.shape[0], w_out), dtype=np.float32)
        hd = self.d // self.heads
        r = hd if self.scheme == "Identity" else self.r  # per head
        check(fn(CODEC_ID[self.scheme], x.shape[0], self.heads, hd, r, _p(self.basis), _p(self.bias),
                 _p(self.kept), _p(x), _p(y)))
        return y

    def encode_vector(self, x):
        return self._call(lib().pikv_codec_encode_host, x, self.d, self.stored_width())[0]

    def decode_vector(self, y):
        return self._call(lib().pikv_codec_decode_host, y, self.stored_width(), self.d)[0]

    def encode(self, key, value):
        return self.encode_vector(key), self.encode_vector(value)

    def decode(self, ck, cv):
        return self.decode_vector(ck), self.decode_vector(cv)

    def reconstruction_error(self, x) -> float:
        x = np.asarray(x, dtype=np.float64)
        n = np.linalg.norm(x)
        if n == 0:
            from .engine import PikvError
            raise PikvError(1, "reconstruction_error: zero-norm input")
        return float(np.linalg.norm(x - self.decode_vector(self.encode_vector(x))) / n)
