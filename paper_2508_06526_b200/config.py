# SPDX-License-Identifier: Apache-2.0
"""Engine configuration mirroring the reference's config structs.

``EngineConfig`` aggregates the same five configs as the reference's
``pikv::EngineConfig`` (pipeline.hpp:87-98): ``ModelConfig`` (config.hpp:23-55),
``StoreConfig`` (kvstore.hpp:63-72), ``RouterConfig`` (router.hpp:24-37),
``SchedulerConfig`` (scheduler.hpp:30-47) and ``CompressorConfig``
(compressor.hpp:28-41), with the reference defaults, plus the B200 runtime
knobs (batch, heads, dtype, ranks).  ``to_c()`` flattens it into the
``pikv_config`` POD of include/pikv_b200.h.
"""
from __future__ import annotations

import ctypes
import dataclasses
from dataclasses import dataclass, field
from typing import List

# ---- enums (same order as the reference) ------------------------------
ROUTER = {"Base": 0, "TopK": 1, "LoadBalanced": 2, "CacheAware": 3, "EntropyLB": 4,
          "Adaptive": 5, "Hierarchical": 6}                      # router.hpp:11-19
SCHED = {"H2O": 0, "SL": 1, "QUEST": 2, "Flex": 3, "LRU": 4, "LRUPlus": 5, "AdaKV": 6,
         "Duo": 7}                                                # scheduler.hpp:16-25
REASON = {0: "budget", 1: "threshold", 2: "overwrite"}             # scheduler.cpp:40-47
CODEC = {"Identity": 0, "LowRank": 1, "SVD": 1, "LoRA": 1, "LoRAPlus": 2, "FastV": 3,
         "Prune": 4, "Int8": 5, "Int4": 6}
DTYPE = {"f32": 0, "bf16": 1}


class PikvConfigC(ctypes.Structure):
    """ctypes image of ``pikv_config`` (include/pikv_b200.h)."""
    _fields_ = [
        ("d", ctypes.c_int32), ("head_width", ctypes.c_int32), ("E", ctypes.c_int32),
        ("k", ctypes.c_int32), ("L", ctypes.c_int64), ("G", ctypes.c_int32),
        ("S", ctypes.c_int32), ("K", ctypes.c_int32), ("elem_bytes", ctypes.c_int32),
        ("rho", ctypes.c_double), ("n_heads", ctypes.c_int32),
        ("n_tok", ctypes.c_int32), ("n_exp", ctypes.c_int32), ("additive", ctypes.c_int32),
        ("shards_per_device", ctypes.c_int32),
        ("router_strategy", ctypes.c_int32), ("groups", ctypes.c_int32),
        ("stride", ctypes.c_int32),
        ("alpha", ctypes.c_double), ("lambda_miss", ctypes.c_double),
        ("beta_ent", ctypes.c_double), ("bandit_step", ctypes.c_double),
        ("bias_cap", ctypes.c_double), ("load_decay", ctypes.c_double),
        ("sched_strategy", ctypes.c_int32), ("budget_pages", ctypes.c_int32),
        ("page_size", ctypes.c_int32), ("sink", ctypes.c_int32),
        ("flex_bucket", ctypes.c_int32), ("n_adakv_weights", ctypes.c_int32),
        ("n_flex_plan", ctypes.c_int32),
        ("tau", ctypes.c_double), ("lambda_freq", ctypes.c_double),
        ("adakv_step", ctypes.c_double), ("target_hit", ctypes.c_double),
        ("gamma_sim", ctypes.c_double), ("theta0", ctypes.c_double),
        ("hit_decay", ctypes.c_double),
        ("adakv_weights", ctypes.c_double * 8), ("flex_plan", ctypes.c_double * 32),
        ("codec", ctypes.c_int32), ("rank", ctypes.c_int32),
        ("unbounded_budget", ctypes.c_int32), ("n_layers", ctypes.c_int32),
        ("batch", ctypes.c_int32), ("kv_dtype", ctypes.c_int32),
        ("world_size", ctypes.c_int32), ("rank_id", ctypes.c_int32),
        ("pool_entries", ctypes.c_int64), ("seed", ctypes.c_uint64),
        ("route_mode", ctypes.c_int32), ("reserved0", ctypes.c_int32),
    ]


@dataclass
class ModelConfig:                      # config.hpp:23-55
    d: int = 64
    head_width: int = 16
    E: int = 8
    k: int = 2
    L: int = 1024
    G: int = 2
    S: int = 16
    K: int = 4
    rho: float = 1.0
    elem_bytes: int = 2

    def d_prime(self) -> int:           # config.hpp:37-40 (round half away from 0)
        x = self.d / self.rho
        dp = int(x + 0.5) if x >= 0 else -int(-x + 0.5)
        return max(1, dp)


@dataclass
class StoreConfig:                      # kvstore.hpp:63-72
    n_tok: int = 64
    n_exp: int = 64
    additive: bool = False
    shards_per_device: int = 0


@dataclass
class RouterConfig:                     # router.hpp:24-37
    strategy: str = "TopK"
    k: int = 2
    alpha: float = 1.0
    lambda_miss: float = 1.0
    beta_ent: float = 1.0
    bandit_step: float = 0.05
    groups: int = 1
    stride: int = 1
    bias_cap: float = 5.0
    load_decay: float = 0.99


@dataclass
class SchedulerConfig:                  # scheduler.hpp:30-47
    strategy: str = "LRU"
    budget_pages: int = 4
    page_size: int = 16
    tau: float = 64.0
    sink: int = 4
    lambda_freq: float = 0.5
    adakv_step: float = 0.05
    target_hit: float = 0.9
    gamma_sim: float = 0.5
    theta0: float = -1e18
    hit_decay: float = 0.9
    adakv_weights: List[float] = field(default_factory=lambda: [1.0, 0.5, 0.25])
    flex_plan: List[float] = field(default_factory=lambda: [1.0])
    flex_bucket: int = 16


@dataclass
class CompressorConfig:                 # compressor.hpp:28-41 (runtime projection part)
    scheme: str = "Identity"
    rank: int = 8


@dataclass
class EngineConfig:                     # pipeline.hpp:87-98
    model: ModelConfig = field(default_factory=ModelConfig)
    store: StoreConfig = field(default_factory=StoreConfig)
    router: RouterConfig = field(default_factory=RouterConfig)
    scheduler: SchedulerConfig = field(default_factory=SchedulerConfig)
    compressor: CompressorConfig = field(default_factory=CompressorConfig)
    unbounded_budget: bool = False
    seed: int = 1
    route_mode: str = "exact"            # "fast": tree-reduced fp64 logits (PIKV_ROUTE_FAST)
    # ---- B200 runtime (no reference counterpart) ----
    n_heads: int = 1
    n_layers: int = 0
    batch: int = 1
    kv_dtype: str = "f32"
    world_size: int = 1
    rank_id: int = 0
    pool_entries: int = 0

    def copy(self) -> "EngineConfig":
        return dataclasses.replace(
            self, model=dataclasses.replace(self.model), store=dataclasses.replace(self.store),
            router=dataclasses.replace(self.router),
            scheduler=dataclasses.replace(
                self.scheduler, adakv_weights=list(self.scheduler.adakv_weights),
                flex_plan=list(self.scheduler.flex_plan)),
            compressor=dataclasses.replace(self.compressor))

    @property
    def head_dim(self) -> int:
        return self.model.d // self.n_heads

    @property
    def stored_per_head(self) -> int:
        if CODEC[self.compressor.scheme] in (1, 2, 3, 4):
            return self.compressor.rank
        return self.head_dim

    @property
    def stored_width(self) -> int:
        return self.stored_per_head * self.n_heads

    def to_c(self) -> PikvConfigC:
        c = PikvConfigC()
        m, s, r, sc = self.model, self.store, self.router, self.scheduler
        c.d, c.head_width, c.E, c.k, c.L = m.d, m.head_width, m.E, r.k, m.L
        c.G, c.S, c.K, c.elem_bytes, c.rho = m.G, m.S, m.K, m.elem_bytes, m.rho
        c.n_heads = self.n_heads
        c.n_tok, c.n_exp, c.additive, c.shards_per_device = (
            s.n_tok, s.n_exp, int(s.additive), s.shards_per_device)
        c.router_strategy, c.groups, c.stride = ROUTER[r.strategy], r.groups, r.stride
        c.alpha, c.lambda_miss, c.beta_ent = r.alpha, r.lambda_miss, r.beta_ent
        c.bandit_step, c.bias_cap, c.load_decay = r.bandit_step, r.bias_cap, r.load_decay
        c.sched_strategy, c.budget_pages, c.page_size = (
            SCHED[sc.strategy], sc.budget_pages, sc.page_size)
        c.sink, c.flex_bucket = sc.sink, sc.flex_bucket
        if len(sc.adakv_weights) > 8 or len(sc.flex_plan) > 32:
            raise ValueError("adakv_weights <= 8 and flex_plan <= 32 entries")
        c.n_adakv_weights, c.n_flex_plan = len(sc.adakv_weights), len(sc.flex_plan)
        for i, w in enumerate(sc.adakv_weights):
            c.adakv_weights[i] = w
        for i, w in enumerate(sc.flex_plan):
            c.flex_plan[i] = w
        c.tau, c.lambda_freq, c.adakv_step = sc.tau, sc.lambda_freq, sc.adakv_step
        c.target_hit, c.gamma_sim, c.theta0, c.hit_decay = (
            sc.target_hit, sc.gamma_sim, sc.theta0, sc.hit_decay)
        c.codec, c.rank = CODEC[self.compressor.scheme], self.compressor.rank
        c.unbounded_budget, c.n_layers = int(self.unbounded_budget), self.n_layers
        c.batch, c.kv_dtype = self.batch, DTYPE[self.kv_dtype]
        c.world_size, c.rank_id, c.pool_entries = self.world_size, self.rank_id, self.pool_entries
        c.seed = self.seed & 0xFFFFFFFFFFFFFFFF
        c.route_mode = {"exact": 0, "fast": 1}[self.route_mode]
        return c
