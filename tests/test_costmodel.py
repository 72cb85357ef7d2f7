# SPDX-License-Identifier: Apache-2.0
"""The analytic cost model: paper_2508_06526_b200.costmodel
against the reference's own costmodel.cpp -- bit-identical doubles on the
golden vectors (tests/golden/make_costmodel_golden.py) -- and the reference's
KATs (test_costmodel.cpp)."""
import json
import math
import os

import numpy as np
import pytest

from paper_2508_06526_b200._capi import PikvError
from paper_2508_06526_b200.config import ModelConfig
from paper_2508_06526_b200.costmodel import (HardwareProfile, cost_report, io_and_roofline,
                                             latency_step, mem_total, mem_total_at,
                                             mem_total_optimal, optimal_shard_size,
                                             optimal_shard_size_of, speedup,
                                             utilization_check)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "costmodel.json")


def flat(r, m):
    """Same order as ref_cost_report (oracle/ref_driver.cpp)."""
    return [r.memory.token, r.memory.page, r.memory.total, r.memory_bytes.token,
            r.memory_bytes.page, r.memory_bytes.total, r.shard.exact,
            float(r.shard.floor_candidate), float(r.shard.ceil_candidate),
            float(r.shard.best_integer), r.shard.best_cost, r.latency.read, r.latency.decode,
            r.latency.step, r.roofline.io_dense, r.roofline.io_sparse, r.roofline.rd_dense,
            r.roofline.rd_sparse, r.roofline.hit_rate, r.roofline.arith_intensity,
            r.roofline.throughput_scaling, 1.0 if r.roofline.compute_bound else 0.0,
            r.utilization.eta_util, r.utilization.threshold, 1.0 if r.utilization.passed else 0.0,
            mem_total_optimal(m), speedup(1.0, m.rho)]


def test_cost_report_matches_reference_bit_for_bit():
    rows = json.load(open(GOLDEN))
    assert len(rows) >= 60
    for c in rows:
        md = dict(c["model"])
        md["rho"] = float.fromhex(md["rho"])
        m = ModelConfig(**md)
        hw = HardwareProfile(*[float.fromhex(x) for x in c["hw"]])
        args = (m, hw, float.fromhex(c["batch"]), c["active"], float.fromhex(c["thr"]))
        if c["rc"]:
            with pytest.raises(PikvError) as ei:
                cost_report(*args)
            assert ei.value.code == c["rc"]
            continue
        got = flat(cost_report(*args), m)
        want = [float.fromhex(x) for x in c["out"]]
        assert [g.hex() for g in got] == [w.hex() for w in want], c["model"]


def cost_config(d, rho, L, G, S, K):  # test_costmodel.cpp:14-26
    return ModelConfig(d=d, head_width=1, rho=rho, L=L, G=G, S=S, K=K, E=8, k=2)


def test_reference_kats():
    m = mem_total(cost_config(64, 2.0, 1024, 4, 8, 2))          # :32-37
    assert (m.token, m.page, m.total) == (64.0 * 32.0, 64.0 * 16.0, 3072.0)
    assert mem_total(cost_config(64, 2.0, 1024, 4, 1, 1)).page == 2.0 * 64.0 / 2.0
    cfg = cost_config(64, 2.0, 1024, 4, 8, 2)
    cfg.elem_bytes = 2
    assert mem_total(cfg, True).total == 2.0 * 3072.0             # :58-62
    s = optimal_shard_size_of(1024.0, 4.0, 16.0)                  # :64-70
    assert math.isclose(s.exact, 4.0) and s.best_integer == 4
    assert math.isclose(optimal_shard_size_of(64.0, 8.0, 8.0).exact, 1.0)
    cfg = cost_config(64, 2.0, 1024, 4, 8, 2)                     # :111-121
    cfg.k = 4
    t = latency_step(cfg, HardwareProfile(1e9, 1e9, 2.0), 1.0)
    assert math.isclose(t.step, 5.12e-7, rel_tol=1e-12) and t.step == t.read + t.decode
    assert speedup(2.0, 4.0) == 2.0 and speedup(3.0, 3.0) == 1.0
    cfg = cost_config(512, 1.0, 4096, 1, 1, 1)                    # :149-175
    cfg.head_width, cfg.E, cfg.k = 64, 64, 4
    r = io_and_roofline(cfg, HardwareProfile(), 1.0)
    assert r.throughput_scaling == 16.0 and math.isclose(r.io_dense / r.io_sparse, 16.0)
    cfg.E = 16
    r = io_and_roofline(cfg, HardwareProfile(), 1.0)
    assert (r.hit_rate, r.rd_dense, r.rd_sparse) == (0.25, 4096.0 / 16.0, 1024.0)
    assert math.isclose(r.arith_intensity, 64.0 / 640.0)
    cfg = cost_config(64, 1.0, 1024, 1, 1, 1)                     # :195-206
    cfg.E, cfg.k = 16, 4
    assert utilization_check(cfg, 16, 0.2).eta_util == 0.25 and utilization_check(cfg, 16, 0.2).passed
    assert utilization_check(cfg, 8, 0.2).eta_util == 0.125 and not utilization_check(cfg, 8, 0.2).passed
    with pytest.raises(PikvError) as ei:
        utilization_check(cfg, 17, 0.2)
    assert ei.value.kind == "InvalidArgument"


def test_reference_error_cases():                                 # :208-216
    cfg = cost_config(64, 2.0, 1024, 4, 8, 2)
    for fn in (lambda: mem_total_at(cfg, 0.0),
               lambda: latency_step(cfg, HardwareProfile(decode_factor=3.0), 1.0),
               lambda: latency_step(cfg, HardwareProfile(), 0.0)):
        with pytest.raises(PikvError) as ei:
            fn()
        assert ei.value.kind == "InvalidConfig"


def test_optimal_shard_substitution():                            # :72-109
    rng = np.random.default_rng(7)
    for _ in range(100):
        cfg = cost_config(int(rng.integers(8, 520)), float(1 + rng.random() * 7),
                          int(rng.integers(1, 100000)), int(rng.integers(1, 17)),
                          int(rng.integers(1, 129)), int(rng.integers(1, 17)))
        closed = optimal_shard_size(cfg)
        grid = [mem_total_at(cfg, float(s)).total for s in range(1, 400)]
        best_s = int(np.argmin(grid)) + 1
        if closed.exact < 398:
            assert abs(best_s - closed.exact) <= 1.0
        assert math.isclose(mem_total_at(cfg, closed.exact).total, mem_total_optimal(cfg),
                            rel_tol=1e-9)
