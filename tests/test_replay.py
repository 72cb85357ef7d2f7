# SPDX-License-Identifier: Apache-2.0
"""Trace replay host logic on CPU: generate_trace and the
PIKT file format against the reference's own trace.cpp (golden fixtures
from tests/golden/make_trace_golden.py), Topology and the runner's
percentile, and the MetricsAccumulator driven by the oracle engine.  The GPU
replay is compared with the oracle replay in test_replay_gpu.py."""
import glob
import json
import os

import numpy as np
import pytest

from oracle_bind import OracleEngine
from paper_2508_06526_b200._capi import PikvError
from paper_2508_06526_b200.replay import (MetricsAccumulator, Topology, Trace, TraceSpec,
                                          generate_trace, load_trace, percentile, save_trace)

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = sorted(glob.glob(os.path.join(HERE, "golden", "trace", "trace_*.npz")))


def spec_of(z):
    steps, width, vocab, skew, _, layers = z["spec"]
    return TraceSpec(int(steps), int(width), int(vocab), float(skew), int(z["seed"]), int(layers))


@pytest.mark.parametrize("path", GOLD)
def test_generate_trace_matches_reference(path):
    z = np.load(path)
    tr = generate_trace(spec_of(z))
    assert np.array_equal(tr.vocabulary, z["vocabulary"])
    assert np.array_equal(tr.embed_ids, z["embed_ids"])
    assert np.array_equal(tr.saliency, z["saliency"])


@pytest.mark.parametrize("path", GOLD)
def test_trace_file_format_matches_reference(path, tmp_path):
    z = np.load(path)
    ref_file = path.replace(".npz", ".pikt")
    tr = load_trace(ref_file)                     # a file the reference wrote
    assert np.array_equal(tr.embed_ids, z["embed_ids"])
    assert np.array_equal(tr.saliency, z["saliency"])
    assert np.array_equal(tr.vocabulary, z["vocabulary"])
    out = tmp_path / "t.pikt"
    save_trace(generate_trace(spec_of(z)), str(out))
    assert out.read_bytes() == open(ref_file, "rb").read()


def test_trace_errors(tmp_path):
    for bad in (TraceSpec(width=0), TraceSpec(vocab=0), TraceSpec(zipf_skew=-1), TraceSpec(layers=0)):
        with pytest.raises(PikvError) as ei:
            generate_trace(bad)
        assert ei.value.kind == "InvalidConfig"
    good = tmp_path / "g.pikt"
    save_trace(generate_trace(TraceSpec(steps=4, width=4, vocab=3)), str(good))
    data = good.read_bytes()
    cases = {"magic": b"XIKT" + data[4:], "version": data[:4] + b"\x02\x00" + data[6:],
             "truncated": data[:-3],
             "range": data[:-(4 + 4 * 4)] + (7).to_bytes(4, "little") + data[-(4 * 4):]}
    for name, blob in cases.items():
        p = tmp_path / (name + ".pikt")
        p.write_bytes(blob)
        with pytest.raises(PikvError) as ei:
            load_trace(str(p))
        assert ei.value.kind == "IoError", name
    with pytest.raises(PikvError):
        load_trace(str(tmp_path / "missing.pikt"))


def test_topology_and_percentile():
    t = Topology.uniform(3, 1e-7, 2e-6, 1e9)
    assert t.fetch_seconds(1, 1, 4096) == 1e-7
    assert t.fetch_seconds(0, 2, 4096) == 2e-6 + 4096 / 1e9
    with pytest.raises(PikvError):
        t.fetch_seconds(3, 0, 1)
    bad = Topology(2, 1e-7, [0.0, 1.0, 2.0, 0.0], [1.0] * 4)
    with pytest.raises(PikvError):
        bad.validate()
    vals = sorted([5.0, 1.0, 3.0, 2.0, 4.0])
    assert [percentile(vals, q) for q in (0.5, 0.95, 0.99)] == [3.0, 5.0, 5.0]
    assert percentile([], 0.5) == 0.0


def oracle_records(cfg, trace):
    """Step records of the oracle engine replaying `trace` (one stream)."""
    orc = OracleEngine(cfg)
    for t in range(trace.spec.steps):
        emb, sal = trace.token(t)
        r = orc.step_embed(emb, sal[:cfg.n_layers] if cfg.n_layers > 0 else None)
        yield {"experts": r["experts"], "gates": list(r["gates"]), "inserts": r["inserts"],
               "fetch_elements": r["fetch_elements"], "hits": r["hits"], "lookups": r["lookups"],
               "att_token": r["att_token"], "att_expert": r["att_expert"],
               "evictions": [e[1:] for e in r["evictions"]],
               "memory_bytes": orc.store_stats()["memory_bytes"]}
    yield orc


def test_metrics_accumulator_on_oracle_replay():
    from cases import engine_config
    cfg = engine_config(router="CacheAware", sched="LRU", d=16, G=4, budget=3, n_layers=4)
    tr = generate_trace(TraceSpec(steps=80, width=16, vocab=24, seed=5, layers=4))
    acc = MetricsAccumulator(cfg, Topology.uniform(4, 1e-7, 2e-6, 1e10), home_device=1,
                             lambda_memory=1e-9, lambda_hit=0.5, seed=5)
    gen = oracle_records(cfg, tr)
    lines = [acc.step(t, next(gen)) for t in range(80)]
    orc = next(gen)
    m = acc.report(orc.router_state()["usage"])
    ev = [json.loads(x) for x in lines]
    assert m["steps"] == 80 and m["fetch_bytes"] == sum(e["fetch_bytes"] for e in ev)
    assert m["hit_rate"] == sum(e["hits"] for e in ev) / sum(e["lookups"] for e in ev)
    reasons = [x["reason"] for e in ev for x in e["evictions"]]
    assert (m["evicted_budget"], m["evicted_overwrite"]) == (reasons.count("budget"),
                                                            reasons.count("overwrite"))
    assert m["latency_total_s"] == pytest.approx(sum(e["latency_s"] for e in ev), rel=1e-12)
    assert m["peak_memory_bytes"] > 0 and sum(m["expert_load"]) == 80 * cfg.router.k
    assert m["objective_value"] == (m["objective_latency_s"] + 1e-9 * m["objective_memory_bytes"]
                                    - 0.5 * m["objective_hit_rate"])


# ------------------------------------ pinned to the reference's runner ----
RUNNER_GOLD = sorted(glob.glob(os.path.join(HERE, "golden", "runner", "*.json")))


def _runner_case(path):
    import sys
    sys.path.insert(0, os.path.join(HERE, "golden"))
    from runner_cases import CASES, LAMBDA_HIT, LAMBDA_MEMORY, LAYERS, TOPO, D
    doc = json.load(open(path))
    c = CASES[doc["case"]]
    spec = TraceSpec(steps=c["T"], width=D, vocab=c["vocab"], zipf_skew=c["skew"], seed=c["tseed"],
                     layers=LAYERS)
    topo = Topology.uniform(c["G"], TOPO["local"], TOPO["link"], TOPO["bw"])
    return doc, c, spec, topo, LAMBDA_MEMORY, LAMBDA_HIT


@pytest.mark.parametrize("path", RUNNER_GOLD, ids=[os.path.basename(p)[:-5] for p in RUNNER_GOLD])
def test_oracle_replay_matches_reference_runner(path):
    """MetricsAccumulator (runner.cpp:69-261 restated) fed by the oracle
    engine reproduces the reference's own run_experiment output byte for
    byte: report line, every event line, the store dump (goldens from
    tests/golden/make_runner_golden.py)."""
    doc, c, spec, topo, lm, lh = _runner_case(path)
    from runner_cases import engine_cfg
    from paper_2508_06526_b200 import wire
    cfg = engine_cfg(c)
    tr = generate_trace(spec)
    acc = MetricsAccumulator(cfg, topo, c["home"], lm, lh, spec.seed)
    gen = oracle_records(cfg, tr)
    lines = [acc.step(t, next(gen)) for t in range(spec.steps)]
    orc = next(gen)
    report = acc.report(orc.router_state()["usage"])
    assert lines == doc["events"]
    assert wire.dumps(report) == doc["report"]
    assert wire.store_dump_lines(orc.snapshot(spec.steps)) == doc["store"]
