# SPDX-License-Identifier: Apache-2.0
"""Configurations of the reference-runner golden runs (trace replay, SURVEY
8 f3): each case is rendered both as the reference's config text
(runconfig.cpp keys, fed to run_experiment by oracle/ref_runner.cpp) and as
this engine's EngineConfig / replay arguments."""

CASES = {
    "topk_lru_g4": dict(router="TopK", sched="LRU", E=8, k=2, G=4, S=64, K=3, n_tok=16, n_exp=8,
                        ps=4, T=60, vocab=20, skew=1.1, tseed=3, seed=7, home=0),
    "adaptive_lruplus_g2": dict(router="Adaptive", sched="LRUPlus", E=8, k=2, G=2, S=32, K=4,
                                n_tok=16, n_exp=8, ps=4, T=70, vocab=24, skew=0.9, tseed=5, seed=11,
                                home=1),
    "hier_sl_e16k4": dict(router="Hierarchical", sched="SL", E=16, k=4, G=4, S=64, K=6, n_tok=4,
                          n_exp=8, ps=4, T=60, vocab=20, skew=1.2, tseed=9, seed=3, home=2,
                          groups=4, tau=20.0),
    "cacheaware_unbounded": dict(router="CacheAware", sched="LRU", E=8, k=2, G=2, S=128, K=4,
                                 n_tok=16, n_exp=8, ps=4, T=50, vocab=16, skew=1.0, tseed=2, seed=5,
                                 home=0, unbounded=True),
    # fp64-mass schedulers: the oracle replay is bit-exact with the reference;
    # the GPU's fp32 attention mass may order pages differently (CPU only)
    "lb_h2o_g2": dict(router="LoadBalanced", sched="H2O", E=8, k=2, G=2, S=32, K=3, n_tok=16,
                      n_exp=8, ps=4, T=60, vocab=20, skew=1.0, tseed=4, seed=9, home=0, cpu_only=True),
    "entropy_duo_g2": dict(router="EntropyLB", sched="Duo", E=8, k=2, G=2, S=32, K=3, n_tok=16,
                           n_exp=8, ps=4, T=60, vocab=20, skew=1.0, tseed=6, seed=13, home=1,
                           cpu_only=True),
}

D, HEAD, LAYERS = 16, 4, 4
TOPO = dict(local=1e-7, link=3e-6, bw=2e10)
LAMBDA_MEMORY, LAMBDA_HIT = 1e-8, 0.25


def config_text(c):
    lines = [
        "model.d = %d" % D, "model.head_width = %d" % HEAD, "model.E = %d" % c["E"],
        "model.k = %d" % c["k"], "model.G = %d" % c["G"], "model.S = %d" % c["S"],
        "model.K = %d" % c["K"], "store.n_tok = %d" % c["n_tok"], "store.n_exp = %d" % c["n_exp"],
        "router.strategy = %s" % c["router"], "router.groups = %d" % c.get("groups", 1),
        "scheduler.strategy = %s" % c["sched"], "scheduler.page_size = %d" % c["ps"],
        "scheduler.tau = %r" % c.get("tau", 64.0),
        "trace.T = %d" % c["T"], "trace.vocab = %d" % c["vocab"], "trace.skew = %r" % c["skew"],
        "trace.seed = %d" % c["tseed"], "trace.layers = %d" % LAYERS,
        "topology.local_latency = %r" % TOPO["local"], "topology.link_latency = %r" % TOPO["link"],
        "topology.link_bandwidth = %r" % TOPO["bw"],
        "objective.lambda_memory = %r" % LAMBDA_MEMORY, "objective.lambda_hit = %r" % LAMBDA_HIT,
        "pipeline.fidelity = false", "pipeline.unbounded = %s" % ("true" if c.get("unbounded") else "false"),
        "run.seed = %d" % c["seed"], "run.home_device = %d" % c["home"], "run.dump_store = store.jsonl",
    ]
    return "\n".join(lines) + "\n"


def engine_cfg(c, batch=1):
    """The same configuration as this engine's EngineConfig (runconfig.cpp's
    derived defaults: L = T, budget = K, rho = d / stored width = 1)."""
    from paper_2508_06526_b200.config import (EngineConfig, ModelConfig, RouterConfig,
                                              SchedulerConfig, StoreConfig)
    e = EngineConfig()
    e.model = ModelConfig(d=D, head_width=HEAD, E=c["E"], k=c["k"], L=c["T"], G=c["G"], S=c["S"],
                          K=c["K"], rho=1.0)
    e.store = StoreConfig(n_tok=c["n_tok"], n_exp=c["n_exp"])
    # runconfig.cpp has no router.k key: routing keeps RouterConfig's k = 2
    # while model.k (the cost model's active experts) follows the config
    e.router = RouterConfig(strategy=c["router"], k=2, groups=c.get("groups", 1))
    e.scheduler = SchedulerConfig(strategy=c["sched"], budget_pages=c["K"], page_size=c["ps"],
                                  tau=c.get("tau", 64.0))
    e.unbounded_budget = bool(c.get("unbounded"))
    e.n_heads, e.n_layers, e.batch, e.kv_dtype, e.seed = 1, LAYERS, batch, "f32", c["seed"]
    return e
