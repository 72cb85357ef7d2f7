# SPDX-License-Identifier: Apache-2.0
"""Shared parity configurations (after test_pipeline.cpp:16-48 engine_config)."""
from paper_2508_06526_b200.config import (CompressorConfig, EngineConfig, ModelConfig,
                                          RouterConfig, SchedulerConfig, StoreConfig)

ROUTERS = ["Base", "TopK", "LoadBalanced", "CacheAware", "EntropyLB", "Adaptive", "Hierarchical"]
SCHEDS = ["H2O", "SL", "Flex", "LRU", "LRUPlus", "AdaKV", "Duo"]


def engine_config(router="TopK", sched="LRU", d=16, E=8, k=2, S=64, G=2, n_tok=16, n_exp=8,
                  budget=4, ps=4, unbounded=False, H=1, n_layers=3, dtype="f32", seed=7,
                  batch=1, codec="Identity", rank=8, theta0=0.5):
    c = EngineConfig()
    c.model = ModelConfig(d=d, head_width=4, E=E, k=k, L=1024, G=G, S=S, K=4, rho=1.0)
    c.store = StoreConfig(n_tok=n_tok, n_exp=n_exp)
    c.router = RouterConfig(strategy=router, k=k, groups=4 if router == "Hierarchical" else 1)
    c.scheduler = SchedulerConfig(strategy=sched, budget_pages=budget, page_size=ps)
    if sched == "AdaKV":
        c.scheduler.theta0 = theta0
    if sched == "Flex":
        c.scheduler.flex_plan = [1.0, 0.5, 0.25, 0.0]
        c.scheduler.flex_bucket = 8
    if sched == "SL":
        c.scheduler.tau = 20.0
    c.compressor = CompressorConfig(scheme=codec, rank=rank)
    c.unbounded_budget = unbounded
    c.n_heads = H
    c.n_layers = n_layers
    c.kv_dtype = dtype
    c.seed = seed
    c.batch = batch
    return c
