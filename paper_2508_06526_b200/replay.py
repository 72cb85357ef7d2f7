# SPDX-License-Identifier: Apache-2.0
"""Trace replay through the engine: the reference's
run_experiment loop (runner.cpp:69-261) over generate_trace inputs
(trace.cpp:54-82), producing the same MetricsReport fields, per-step event
lines (runner.cpp:183-196) and final store dump (runner.cpp:215-222).

* ``generate_trace`` runs in libpikv_b200 (the reference's Rng); traces
  round-trip through the reference's PIKT v1 file format (trace.cpp:84-134).
* ``Topology`` (topology.hpp:13-78) prices each attended entry's fetch.
* ``MetricsAccumulator`` consumes one step record per step (experts, gates,
  inserts, fetch_elements, hits, lookups, attended (token, expert) in the
  reference's retrieval order, eviction records, store memory bytes) and
  finishes with runner.cpp's aggregates; ``run_trace`` feeds it from the GPU
  engine (one stream per trace, ``Engine.step_embed_host``).
Fidelity (the ReferenceDecoder comparison, runner.cpp:158-162) is not
recomputed: ``fidelity_enabled`` is false and each step's fidelity is 0.0.
"""
from __future__ import annotations

import ctypes
import math
import struct
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from . import wire
from ._capi import PikvError, check, lib
from .config import EngineConfig
from .costmodel import HardwareProfile, io_and_roofline, mem_total, optimal_shard_size

INVALID_ARGUMENT, INVALID_CONFIG, IO_ERROR = 1, 2, 9


@dataclass
class TraceSpec:                        # trace.hpp:12-21
    steps: int = 256
    width: int = 16
    vocab: int = 64
    zipf_skew: float = 1.0
    seed: int = 1
    layers: int = 4

    def validate(self) -> None:         # trace.cpp:39-44
        if self.width < 1:
            raise PikvError(INVALID_CONFIG, "TraceSpec: width must be >= 1")
        if self.vocab < 1:
            raise PikvError(INVALID_CONFIG, "TraceSpec: vocab must be >= 1")
        if self.zipf_skew < 0:
            raise PikvError(INVALID_CONFIG, "TraceSpec: skew must be >= 0")
        if self.layers < 1:
            raise PikvError(INVALID_CONFIG, "TraceSpec: layers must be >= 1")


@dataclass
class Trace:                            # trace.hpp:28-36
    spec: TraceSpec
    vocabulary: np.ndarray              # [vocab][width] fp64
    embed_ids: np.ndarray               # [steps] uint32
    saliency: np.ndarray                # [steps][layers] fp32

    def token(self, i: int):
        """Trace::token (trace.cpp:46-52): (embedding, layer_saliency)."""
        return self.vocabulary[self.embed_ids[i]], self.saliency[i].astype(np.float64)


def _gen(spec: TraceSpec, want_events: bool):
    spec.validate()
    voc = np.zeros((spec.vocab, spec.width), dtype=np.float64)
    ids = np.zeros(max(spec.steps, 1), dtype=np.uint32)
    sal = np.zeros((max(spec.steps, 1), spec.layers), dtype=np.float32)
    check(lib().pikv_generate_trace(spec.steps, spec.width, spec.vocab, spec.zipf_skew, spec.seed,
                                    spec.layers, voc.ctypes.data,
                                    ids.ctypes.data if want_events else None,
                                    sal.ctypes.data if want_events else None))
    return voc, ids[:spec.steps], sal[:spec.steps]


def generate_trace(spec: TraceSpec) -> Trace:
    """trace.cpp:54-82."""
    voc, ids, sal = _gen(spec, True)
    return Trace(spec, voc, ids, sal)


_MAGIC, _VERSION = b"PIKT", 1


def save_trace(trace: Trace, path: str) -> None:
    """trace.cpp:84-98: header + per step (embed id, layer saliency)."""
    s = trace.spec
    try:
        with open(path, "wb") as f:
            f.write(_MAGIC + struct.pack("<HQIIdQI", _VERSION, s.steps, s.width, s.vocab, s.zipf_skew,
                                         s.seed, s.layers))
            for t in range(s.steps):
                f.write(struct.pack("<I", int(trace.embed_ids[t])))
                f.write(np.ascontiguousarray(trace.saliency[t], dtype="<f4").tobytes())
    except OSError as ex:
        raise PikvError(IO_ERROR, "trace save: cannot open %s (%s)" % (path, ex))


def load_trace(path: str) -> Trace:
    """trace.cpp:100-132; the vocabulary is regenerated from the spec."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise PikvError(IO_ERROR, "trace load: cannot open " + path)
    if data[:4] != _MAGIC:
        raise PikvError(IO_ERROR, "trace load: bad magic")
    off = 4

    def take(fmt):
        nonlocal off
        n = struct.calcsize(fmt)
        if off + n > len(data):
            raise PikvError(IO_ERROR, "trace file truncated")
        v = struct.unpack_from(fmt, data, off)
        off += n
        return v

    if take("<H")[0] != _VERSION:
        raise PikvError(IO_ERROR, "trace load: unsupported version")
    steps, width, vocab, skew, seed, layers = take("<QIIdQI")
    spec = TraceSpec(steps, width, vocab, skew, seed, layers)
    voc, _, _ = _gen(spec, False)
    ids = np.zeros(steps, dtype=np.uint32)
    sal = np.zeros((steps, layers), dtype=np.float32)
    for t in range(steps):
        ids[t] = take("<I")[0]
        if ids[t] >= vocab:
            raise PikvError(IO_ERROR, "trace load: embed id out of range")
        sal[t] = take("<%df" % layers)
    return Trace(spec, voc, ids, sal)


@dataclass
class Topology:                         # topology.hpp:13-78
    devices: int = 1
    local_latency: float = 1e-7
    link_latency: List[float] = field(default_factory=lambda: [0.0])
    link_bandwidth: List[float] = field(default_factory=lambda: [1.0])

    @staticmethod
    def uniform(devices: int, local_latency: float, link_latency: float,
                link_bandwidth: float) -> "Topology":
        lat = [0.0 if i == j else link_latency for i in range(devices) for j in range(devices)]
        t = Topology(devices, local_latency, lat, [link_bandwidth] * devices * devices)
        t.validate()
        return t

    def validate(self) -> None:
        G = self.devices
        if G < 1:
            raise PikvError(INVALID_CONFIG, "Topology: devices must be >= 1")
        if len(self.link_latency) != G * G or len(self.link_bandwidth) != G * G:
            raise PikvError(INVALID_CONFIG, "Topology: matrix size mismatch")
        if self.local_latency < 0:
            raise PikvError(INVALID_CONFIG, "Topology: negative local latency")
        for i in range(G):
            for j in range(G):
                if self.link_latency[i * G + j] != self.link_latency[j * G + i]:
                    raise PikvError(INVALID_CONFIG, "Topology: latency matrix not symmetric")
                if i == j and self.link_latency[i * G + j] != 0.0:
                    raise PikvError(INVALID_CONFIG, "Topology: nonzero diagonal latency")
                if self.link_bandwidth[i * G + j] <= 0.0:
                    raise PikvError(INVALID_CONFIG, "Topology: bandwidth must be positive")

    def fetch_seconds(self, src: int, dst: int, nbytes: int) -> float:
        if src < 0 or src >= self.devices or dst < 0 or dst >= self.devices:
            raise PikvError(INVALID_ARGUMENT, "fetch: device index out of range")
        if src == dst:
            return self.local_latency
        idx = src * self.devices + dst
        return self.link_latency[idx] + float(nbytes) / self.link_bandwidth[idx]


def percentile(sorted_values: Sequence[float], q: float) -> float:
    """runner.cpp:19-26."""
    if not len(sorted_values):
        return 0.0
    idx = int(math.ceil(q * float(len(sorted_values))))
    if idx > 0:
        idx -= 1
    return sorted_values[min(idx, len(sorted_values) - 1)]


def shard_devices(tokens, experts, cfg: EngineConfig) -> np.ndarray:
    """KVStore::locate(token, expert).device (kvstore.cpp:14-30, 102-105) for
    the runner's latency pricing, which the reference also does on the host:
    raw = (t mod n_tok) XOR (or +) (e mod n_exp), device = raw mod G (the
    moduli are powers of two, validated at engine creation)."""
    t = np.asarray(tokens, dtype=np.int64)
    e = np.asarray(experts, dtype=np.int64)
    lhs, rhs = t % cfg.store.n_tok, e % cfg.store.n_exp
    raw = lhs + rhs if cfg.store.additive else lhs ^ rhs
    return (raw % cfg.model.G).astype(np.int32)


class MetricsAccumulator:
    """run_experiment's per-step accounting and final report (runner.cpp:91-261)."""

    def __init__(self, cfg: EngineConfig, topology: Topology, home_device: int = 0,
                 lambda_memory: float = 0.0, lambda_hit: float = 0.0, seed: int = 0,
                 hardware: HardwareProfile | None = None, batch_tokens: float = 1.0):
        self.cfg, self.topo, self.home = cfg, topology, home_device
        self.lambda_memory, self.lambda_hit, self.seed = lambda_memory, lambda_hit, seed
        self.hw = hardware or HardwareProfile()
        self.batch_tokens = batch_tokens
        d_stored = cfg.stored_width
        self.d_stored = d_stored
        self.head = min(cfg.model.head_width, d_stored)
        self.entry_bytes = (2 * self.head + d_stored) * cfg.model.elem_bytes
        self.lat: List[float] = []
        self.latency_total = 0.0
        self.fetch_bytes = 0
        self.io_measured = 0.0
        self.hits = self.lookups = self.retrieved = 0
        self.peak_memory = 0
        self.ev = {0: 0, 1: 0, 2: 0}
        self.events: List[str] = []

    def step(self, t: int, rec: dict) -> str:
        """One step record -> the event line; rec: experts, gates, inserts,
        fetch_elements, hits, lookups, att_token, att_expert ((token,
        expert) order), evictions [(id, token, expert, device, score,
        reason)], memory_bytes."""
        lat = 0.0
        devs = shard_devices(rec["att_token"], rec["att_expert"], self.cfg)
        for dv in devs:  # runner.cpp:105-109, in retrieval order
            lat += self.topo.fetch_seconds(int(dv), self.home, self.entry_bytes)
        misses = rec["lookups"] - rec["hits"]
        if misses > 0 and self.cfg.model.G > 1:  # :110-118
            neighbor = (self.home + 1) % self.cfg.model.G
            lat += float(misses) * self.topo.fetch_seconds(neighbor, self.home, self.entry_bytes)
        elif misses > 0:
            lat += float(misses) * self.topo.local_latency
        self.lat.append(lat)
        self.latency_total += lat
        fb = int(rec["fetch_elements"]) * self.cfg.model.elem_bytes
        self.fetch_bytes += fb
        self.io_measured += float(rec["fetch_elements"])
        self.hits += rec["hits"]
        self.lookups += rec["lookups"]
        self.retrieved += len(rec["att_token"])
        self.peak_memory = max(self.peak_memory, int(rec["memory_bytes"]))
        for ev in rec["evictions"]:
            self.ev[int(ev[5])] += 1
        line = wire.step_event_line(t, rec["experts"], rec["gates"], rec["inserts"], fb, rec["hits"],
                                    rec["lookups"], lat, 0.0, rec["evictions"])
        self.events.append(line)
        return line

    def report(self, expert_load) -> dict:
        """runner.cpp:166-223 aggregates + the report object (:224-259)."""
        cfg, m = self.cfg, self.cfg.model
        steps = len(self.lat)
        hit_rate = 0.0 if self.lookups == 0 else float(self.hits) / float(self.lookups)
        lat_sorted = sorted(self.lat)
        mean = self.latency_total / len(self.lat) if self.lat else 0.0
        roof = io_and_roofline(m, self.hw, self.batch_tokens)
        mean_prefix = (0.0 if self.lookups == 0 else
                       float(self.retrieved) / float(m.k) / float(steps))
        # runner.cpp:236-241 divides and multiplies by the MODEL's k (the
        # cost model's active experts), not the router's
        io_model = (2.0 * self.head + self.d_stored) * mean_prefix * m.k * float(steps)
        obj_lat, obj_mem, obj_hit = self.latency_total, float(self.peak_memory), hit_rate
        return {
            "type": "metrics", "steps": steps, "seed": self.seed,
            "router": cfg.router.strategy, "scheduler": cfg.scheduler.strategy,
            "compressor": cfg.compressor.scheme,
            "hit_rate": hit_rate, "local_fetch_fraction": hit_rate,
            "latency_total_s": self.latency_total, "latency_mean_s": mean,
            "latency_p50_s": percentile(lat_sorted, 0.50),
            "latency_p95_s": percentile(lat_sorted, 0.95),
            "latency_p99_s": percentile(lat_sorted, 0.99),
            "fetch_bytes": self.fetch_bytes, "peak_memory_bytes": self.peak_memory,
            "fidelity_enabled": False, "fidelity_cumulative": 0.0,
            "expert_load": [int(x) for x in expert_load],
            "evicted_budget": self.ev[0], "evicted_threshold": self.ev[1],
            "evicted_overwrite": self.ev[2],
            "objective_latency_s": obj_lat, "objective_memory_bytes": obj_mem,
            "objective_hit_rate": obj_hit, "lambda_memory": self.lambda_memory,
            "lambda_hit": self.lambda_hit,
            "objective_value": obj_lat + self.lambda_memory * obj_mem - self.lambda_hit * obj_hit,
            "throughput_scaling": roof.throughput_scaling, "hit_rate_model": roof.hit_rate,
            "arith_intensity": roof.arith_intensity,
            "mem_model_total_bytes": mem_total(m, True).total,
            "shard_size_opt": optimal_shard_size(m).exact,
            "io_measured_elements": self.io_measured, "io_model_elements": io_model,
            "io_model_ratio": 1.0 if io_model == 0.0 else self.io_measured / io_model,
        }


@dataclass
class RunOutput:                        # runner.hpp:58-63
    metrics: dict
    report_line: str
    event_log: List[str]
    store_dump: List[str]


def engine_step_records(eng, B: int):
    """The last step of every stream as MetricsAccumulator records."""
    experts, gates, _, summ = eng.read_step()
    evs = eng.read_evictions()
    out = []
    for s in range(B):
        tok, ex, _ = eng.read_attended(s)
        order = np.lexsort((ex, tok))  # KVStore::retrieve order (kvstore.cpp:144-163)
        out.append({
            "experts": [int(x) for x in experts[s]], "gates": [float(g) for g in gates[s]],
            "inserts": int(summ[s]["inserts"]), "fetch_elements": int(summ[s]["fetch_elements"]),
            "hits": int(summ[s]["hits"]), "lookups": int(summ[s]["lookups"]),
            "att_token": tok[order], "att_expert": ex[order],
            "evictions": [(e.entry_id, e.token_id, e.expert_id, e.device, e.score,
                           {"budget": 0, "threshold": 1, "overwrite": 2}[e.reason])
                          for e in evs if e.stream == s],
            "memory_bytes": int(eng.store_stats(s)["memory_bytes"]),
        })
    return out


def run_trace(cfg: EngineConfig, traces: Sequence[Trace], topology: Topology | None = None,
              home_device: int = 0, lambda_memory: float = 0.0, lambda_hit: float = 0.0,
              dump_store: bool = False, hardware: HardwareProfile | None = None,
              batch_tokens: float = 1.0) -> List[RunOutput]:
    """run_experiment (runner.cpp:69-261) on the GPU engine: stream s of a
    cfg.batch-stream engine replays traces[s] (same steps and width)."""
    from .engine import Engine
    B = cfg.batch
    if len(traces) != B:
        raise PikvError(INVALID_ARGUMENT, "run_trace: one trace per stream")
    steps = traces[0].spec.steps
    if any(t.spec.steps != steps or t.spec.width != cfg.model.d for t in traces):
        raise PikvError(INVALID_ARGUMENT, "run_trace: traces need equal steps and width d")
    topo = topology or Topology.uniform(cfg.model.G, 1e-7, 0.0, 1.0)
    accs = [MetricsAccumulator(cfg, topo, home_device, lambda_memory, lambda_hit,
                               traces[s].spec.seed, hardware, batch_tokens) for s in range(B)]
    eng = Engine(cfg)
    try:
        for t in range(steps):
            emb = np.stack([tr.token(t)[0] for tr in traces])
            sal = (np.stack([tr.token(t)[1][:cfg.n_layers] for tr in traces])
                   if cfg.n_layers > 0 else None)
            eng.step_embed_host(emb, sal)
            for s, rec in enumerate(engine_step_records(eng, B)):
                accs[s].step(t, rec)
        outs = []
        for s in range(B):
            metrics = accs[s].report(eng.router_state(s)["usage"])
            dump = wire.store_dump_lines(eng.snapshot(s, steps)) if dump_store else []
            outs.append(RunOutput(metrics, wire.dumps(metrics), list(accs[s].events), dump))
        return outs
    finally:
        eng.close()
