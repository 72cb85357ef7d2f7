# SPDX-License-Identifier: Apache-2.0
"""Config validation of the C-ABI (no GPU needed: pikv_engine_create checks
the configuration before any CUDA call).  Each case is a reference validate()
rule: ModelConfig (config.hpp:42-54), StoreConfig (kvstore.cpp:56-64),
RouterConfig (router.cpp:40-53), SchedulerConfig (scheduler.cpp:49-71), plus
QUEST without a fitted scorer -> NotFitted (scheduler.cpp:199-203)."""
import ctypes

import pytest

from cases import engine_config
from paper_2508_06526_b200 import _capi

L = _capi.lib()


def create_rc(cfg):
    c = cfg.to_c()
    h = ctypes.c_void_p()
    rc = L.pikv_engine_create(ctypes.byref(c), 0, ctypes.byref(h))
    if rc == 0:
        L.pikv_engine_destroy(h)
    return rc


def mutate(**kw):
    cfg = engine_config()
    for path, val in kw.items():
        obj = cfg
        parts = path.split("__")
        for p in parts[:-1]:
            obj = getattr(obj, p)
        setattr(obj, parts[-1], val)
    return cfg


@pytest.mark.parametrize("kw", [
    dict(model__d=0), dict(model__head_width=0), dict(model__head_width=17), dict(model__E=0),
    dict(router__k=0), dict(router__k=9), dict(model__L=0), dict(model__G=0), dict(model__S=0),
    dict(model__K=0), dict(model__rho=0.5), dict(model__elem_bytes=0),
    dict(store__n_tok=3), dict(store__n_exp=6), dict(store__shards_per_device=-1),
    dict(router__alpha=-1.0), dict(router__groups=0), dict(router__groups=9),
    dict(router__load_decay=1.0), dict(scheduler__budget_pages=0), dict(scheduler__page_size=0),
    dict(scheduler__lambda_freq=-0.1), dict(scheduler__target_hit=1.5),
    dict(scheduler__hit_decay=1.0), dict(scheduler__flex_plan=[]), dict(scheduler__sink=-1),
    dict(n_heads=3),
])
def test_invalid_config_rejected(kw):
    assert create_rc(mutate(**kw)) == 2  # PIKV_ERR_INVALID_CONFIG


def test_quest_without_fit_is_not_fitted():
    assert create_rc(engine_config(sched="QUEST")) == 6  # PIKV_ERR_NOT_FITTED


def test_error_message_names_the_rule():
    create_rc(mutate(store__n_tok=3))
    assert b"powers of two" in L.pikv_last_error()


def test_shard_assign_host_validation_without_gpu():
    d = ctypes.c_int32()
    t = ctypes.c_int64(5)
    e = ctypes.c_int32(3)
    rc = L.pikv_shard_assign_host(ctypes.byref(t), ctypes.byref(e), 1, 3, 4, 2, 0,
                                  ctypes.byref(d), None, None)
    assert rc == 2  # kvstore.cpp:17-19


def group_rc(cfg, n_micro):
    c = cfg.to_c()
    h = ctypes.c_void_p()
    rc = L.pikv_group_create(ctypes.byref(c), n_micro, 0, 0, ctypes.byref(h))
    if rc == 0:
        L.pikv_group_destroy(h)
    return rc


@pytest.mark.parametrize("batch,n_micro,world,rank", [(3, 2, 1, 0), (4, 0, 1, 0), (4, 3, 1, 0),
                                                     (4, 2, 2, 2)])
def test_group_rejects_bad_split_before_cuda(batch, n_micro, world, rank):
    """pikv_group_create: the batch must split evenly into n_micro >= 1
    micro-batches, and rank_id < world_size -> InvalidConfig, checked before
    any CUDA call (include/pikv_b200.h, micro-batch pipeline)."""
    cfg = engine_config(batch=batch)
    cfg.world_size, cfg.rank_id = world, rank
    assert _capi.ERRORS[group_rc(cfg, n_micro)] == "InvalidConfig"


def test_group_rejects_invalid_engine_config():
    cfg = mutate(model__d=0)
    cfg.batch = 2
    assert _capi.ERRORS[group_rc(cfg, 2)] == "InvalidConfig"
