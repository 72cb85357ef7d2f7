# SPDX-License-Identifier: Apache-2.0
"""Trace replay on the GPU: run_trace (generate_trace ->
Engine.step_embed_host -> runner.cpp's MetricsReport, event log, store dump)
against the same accumulator fed by the oracle engine.  Everything is
identical except the gates in the event lines (rel 1e-12: CUDA vs glibc
exp).  Schedulers whose scores are integers (LRU, LRU+, SL): replay cannot
inject the oracle's attention mass, which H2O/AdaKV/Duo score by."""
import json

import numpy as np
import pytest

from cases import engine_config
from oracle_bind import OracleEngine
from test_replay import oracle_records

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2508_06526_b200 import wire  # noqa: E402
from paper_2508_06526_b200.replay import (MetricsAccumulator, Topology, TraceSpec,  # noqa: E402
                                          generate_trace, run_trace)


@pytest.mark.parametrize("router,sched,kw", [
    ("TopK", "LRU", dict(G=4, budget=3)),
    ("Adaptive", "LRUPlus", dict(G=2, budget=4, H=2)),
    ("Hierarchical", "SL", dict(E=16, k=4, G=4, n_tok=4, n_exp=8)),
])
def test_run_trace_matches_oracle_replay(router, sched, kw):
    cfg = engine_config(router=router, sched=sched, d=16, batch=2, n_layers=4, **kw)
    traces = [generate_trace(TraceSpec(steps=60, width=16, vocab=20, zipf_skew=1.1, seed=s + 3,
                                       layers=4)) for s in range(2)]
    topo = Topology.uniform(cfg.model.G, 1e-7, 3e-6, 2e10)
    outs = run_trace(cfg, traces, topo, home_device=0, lambda_memory=1e-8, lambda_hit=0.25,
                     dump_store=True)
    for s, tr in enumerate(traces):
        c1 = engine_config(router=router, sched=sched, d=16, batch=1, n_layers=4, **kw)
        acc = MetricsAccumulator(c1, topo, 0, 1e-8, 0.25, tr.spec.seed)
        gen = oracle_records(c1, tr)
        want_lines = [acc.step(t, next(gen)) for t in range(tr.spec.steps)]
        orc = next(gen)
        want = acc.report(orc.router_state()["usage"])
        got = outs[s].metrics
        assert got.keys() == want.keys()
        for key in want:
            assert got[key] == want[key], (s, key, got[key], want[key])
        assert outs[s].report_line == wire.dumps(want)
        for a, b in zip(outs[s].event_log, want_lines):
            ja, jb = json.loads(a), json.loads(b)
            ga, gb = ja.pop("gates"), jb.pop("gates")
            assert ja == jb
            assert np.allclose(ga, gb, rtol=1e-12, atol=0)
        assert outs[s].store_dump == wire.store_dump_lines(orc.snapshot(tr.spec.steps))


# ------------------------------------ pinned to the reference's runner ----
import glob  # noqa: E402
import os  # noqa: E402
import sys  # noqa: E402

_HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(_HERE, "golden"))
from runner_cases import CASES  # noqa: E402

_GPU_CASES = [p for p in sorted(glob.glob(os.path.join(_HERE, "golden", "runner", "*.json")))
              if not CASES[os.path.basename(p)[:-5]].get("cpu_only")]


@pytest.mark.parametrize("path", _GPU_CASES, ids=[os.path.basename(p)[:-5] for p in _GPU_CASES])
def test_run_trace_matches_reference_runner(path):
    """run_trace on the GPU == the reference's own run_experiment output
    (tests/golden/runner, from tests/golden/make_runner_golden.py): report
    line and store dump byte for byte, event lines byte for byte except the
    gates (rel 1e-12: CUDA vs glibc exp)."""
    from runner_cases import engine_cfg
    from test_replay import _runner_case
    doc, c, spec, topo, lm, lh = _runner_case(path)
    out = run_trace(engine_cfg(c), [generate_trace(spec)], topo, home_device=c["home"], lambda_memory=lm,
                    lambda_hit=lh, dump_store=True)[0]
    assert out.report_line == doc["report"]
    assert out.store_dump == doc["store"]
    assert len(out.event_log) == len(doc["events"])
    for a, b in zip(out.event_log, doc["events"]):
        ja, jb = json.loads(a), json.loads(b)
        ga, gb = ja.pop("gates"), jb.pop("gates")
        assert ja == jb
        assert np.allclose(ga, gb, rtol=1e-12, atol=0)
