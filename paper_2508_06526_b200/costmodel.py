# SPDX-License-Identifier: Apache-2.0
"""The reference's analytic cost model (costmodel.hpp / costmodel.cpp),
printed by bench.py beside the measurements.

Host arithmetic only: every formula keeps the reference's operation order so
the doubles are identical (tests/test_costmodel.py checks them against the
reference's own costmodel.cpp compiled into oracle/_ref).  Units follow the
reference: memory in elements (x elem_bytes when in_bytes), I/O in
elements, latencies in seconds, rates in bytes/s and FLOP/s.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

from ._capi import PikvError
from .config import ModelConfig

INVALID_ARGUMENT, INVALID_CONFIG = 1, 2


def validate_model(cfg: ModelConfig) -> None:
    """ModelConfig::validate (config.hpp:42-55)."""
    checks = [(cfg.d < 1, "d must be >= 1"),
              (cfg.head_width < 1 or cfg.head_width > cfg.d, "head_width must be in [1, d]"),
              (cfg.E < 1, "E must be >= 1"), (cfg.k < 1 or cfg.k > cfg.E, "need 1 <= k <= E"),
              (cfg.L < 1, "L must be >= 1"), (cfg.G < 1, "G must be >= 1"),
              (cfg.S < 1, "S must be >= 1"), (cfg.K < 1, "K must be >= 1"),
              (not (cfg.rho >= 1.0), "rho must be >= 1"),
              (cfg.elem_bytes < 1, "elem_bytes must be >= 1")]
    for bad, msg in checks:
        if bad:
            raise PikvError(INVALID_CONFIG, "ModelConfig: " + msg)


@dataclass
class HardwareProfile:                  # costmodel.hpp:11-27
    hbm_bandwidth: float = 1e9          # beta, bytes/s
    core_throughput: float = 1e9        # gamma, bytes/s
    decode_factor: float = 1.0          # eta, in (0, 2]
    peak_compute: float = 1e12          # FLOP/s
    peak_mem_bw: float = 1e11           # bytes/s

    def validate(self) -> None:
        if (self.hbm_bandwidth <= 0 or self.core_throughput <= 0 or self.peak_compute <= 0
                or self.peak_mem_bw <= 0):
            raise PikvError(INVALID_CONFIG, "HardwareProfile: rates must be positive")
        if self.decode_factor <= 0 or self.decode_factor > 2.0:
            raise PikvError(INVALID_CONFIG, "HardwareProfile: decode factor must be in (0, 2]")


@dataclass
class MemoryBreakdown:                  # costmodel.hpp:38-42
    token: float = 0.0
    page: float = 0.0
    total: float = 0.0


@dataclass
class OptimalShardSize:                 # costmodel.hpp:54-60
    exact: float = 0.0
    floor_candidate: int = 1
    ceil_candidate: int = 1
    best_integer: int = 1
    best_cost: float = 0.0


@dataclass
class StepLatency:                      # costmodel.hpp:76-80
    read: float = 0.0
    decode: float = 0.0
    step: float = 0.0


@dataclass
class IoRoofline:                       # costmodel.hpp:93-102
    io_dense: float = 0.0
    io_sparse: float = 0.0
    rd_dense: float = 0.0
    rd_sparse: float = 0.0
    hit_rate: float = 0.0
    arith_intensity: float = 0.0
    throughput_scaling: float = 0.0
    compute_bound: bool = False


@dataclass
class UtilizationCheck:                 # costmodel.hpp:108-112
    eta_util: float = 0.0
    threshold: float = 0.0
    passed: bool = False


@dataclass
class CostReport:                       # costmodel.hpp:118-125
    memory: MemoryBreakdown = field(default_factory=MemoryBreakdown)
    memory_bytes: MemoryBreakdown = field(default_factory=MemoryBreakdown)
    shard: OptimalShardSize = field(default_factory=OptimalShardSize)
    latency: StepLatency = field(default_factory=StepLatency)
    roofline: IoRoofline = field(default_factory=IoRoofline)
    utilization: UtilizationCheck = field(default_factory=UtilizationCheck)


def mem_total_at(cfg: ModelConfig, shard_size: float, in_bytes: bool = False) -> MemoryBreakdown:
    """costmodel.cpp:8-23: M_token = (2d/rho) L/(G S), M_page = (2d/rho) K S."""
    if shard_size <= 0.0:
        raise PikvError(INVALID_CONFIG, "mem_total: shard size must be positive")
    validate_model(cfg)
    two_dp = 2.0 * cfg.d / cfg.rho
    scale = float(cfg.elem_bytes) if in_bytes else 1.0
    m = MemoryBreakdown()
    m.token = scale * two_dp * float(cfg.L) / (float(cfg.G) * shard_size)
    m.page = scale * two_dp * float(cfg.K) * shard_size
    m.total = m.token + m.page
    return m


def mem_total(cfg: ModelConfig, in_bytes: bool = False) -> MemoryBreakdown:
    """costmodel.cpp:25-28."""
    return mem_total_at(cfg, float(cfg.S), in_bytes)


def optimal_shard_size_of(tokens: float, pages: float, devices: float) -> OptimalShardSize:
    """costmodel.cpp:30-48: S* = sqrt(L / (K G)) and the better integer."""
    if tokens <= 0 or pages <= 0 or devices <= 0:
        raise PikvError(INVALID_CONFIG, "optimal_shard_size: parameters must be positive")
    out = OptimalShardSize()
    out.exact = math.sqrt(tokens / (pages * devices))
    out.floor_candidate = max(1, int(math.floor(out.exact)))
    out.ceil_candidate = max(1, int(math.ceil(out.exact)))

    def cost(s):
        return tokens / (devices * s) + pages * s

    fc, cc = cost(float(out.floor_candidate)), cost(float(out.ceil_candidate))
    out.best_integer = out.floor_candidate if fc <= cc else out.ceil_candidate
    out.best_cost = min(fc, cc)
    return out


def optimal_shard_size(cfg: ModelConfig) -> OptimalShardSize:
    """costmodel.cpp:50-56 (cost scaled to element units)."""
    out = optimal_shard_size_of(float(cfg.L), float(cfg.K), float(cfg.G))
    out.best_cost *= 2.0 * cfg.d / cfg.rho
    return out


def mem_total_optimal(cfg: ModelConfig) -> float:
    """costmodel.cpp:58-62: M* = (4d/rho) sqrt(K L / G)."""
    return 4.0 * cfg.d / cfg.rho * math.sqrt(float(cfg.K) * float(cfg.L) / float(cfg.G))


def latency_step(cfg: ModelConfig, hw: HardwareProfile, batch_tokens: float) -> StepLatency:
    """costmodel.cpp:64-78: T_read = 2 d' k B / beta, T_decode = eta d' k B / gamma."""
    validate_model(cfg)
    hw.validate()
    if batch_tokens <= 0:
        raise PikvError(INVALID_CONFIG, "latency_step: batch must be positive")
    dp = cfg.d / cfg.rho
    t = StepLatency()
    t.read = 2.0 * dp * cfg.k * batch_tokens / hw.hbm_bandwidth
    t.decode = hw.decode_factor * dp * cfg.k * batch_tokens / hw.core_throughput
    t.step = t.read + t.decode
    return t


def speedup(rho_from: float, rho_to: float) -> float:
    """costmodel.cpp:80-85."""
    if rho_from <= 0 or rho_to <= 0:
        raise PikvError(INVALID_CONFIG, "speedup: ratios must be positive")
    return rho_to / rho_from


def io_and_roofline(cfg: ModelConfig, hw: HardwareProfile, batch_tokens: float) -> IoRoofline:
    """costmodel.cpp:87-107: dense/sparse I/O (elements), reuse distance,
    hit rate k/E, arithmetic intensity h/(2h+d), roofline scaling E/k."""
    validate_model(cfg)
    hw.validate()
    B, L, h, d = batch_tokens, float(cfg.L), float(cfg.head_width), float(cfg.d)
    E, k = float(cfg.E), float(cfg.k)
    r = IoRoofline()
    r.io_dense = 2.0 * B * L * h * E + B * L * d * E
    r.io_sparse = 2.0 * B * L * h * k + B * L * d * k
    r.rd_dense = L / E
    r.rd_sparse = L / k
    r.hit_rate = k / E
    r.arith_intensity = h / (2.0 * h + d)
    r.throughput_scaling = E / k
    r.compute_bound = r.arith_intensity * hw.peak_mem_bw >= hw.peak_compute
    return r


def utilization_check(cfg: ModelConfig, active_experts: int, threshold: float) -> UtilizationCheck:
    """costmodel.cpp:109-121: eta_util = (k/E) (active/E)."""
    validate_model(cfg)
    if active_experts < 0 or active_experts > cfg.E:
        raise PikvError(INVALID_ARGUMENT, "utilization_check: active count outside [0, E]")
    u = UtilizationCheck()
    u.threshold = threshold
    u.eta_util = (float(cfg.k) / cfg.E) * (float(active_experts) / cfg.E)
    u.passed = u.eta_util >= threshold
    return u


def cost_report(cfg: ModelConfig, hw: HardwareProfile, batch_tokens: float, active_experts: int,
                util_threshold: float) -> CostReport:
    """costmodel.cpp:123-135."""
    r = CostReport()
    r.memory = mem_total(cfg, False)
    r.memory_bytes = mem_total(cfg, True)
    r.shard = optimal_shard_size(cfg)
    r.latency = latency_step(cfg, hw, batch_tokens)
    r.roofline = io_and_roofline(cfg, hw, batch_tokens)
    r.utilization = utilization_check(cfg, active_experts, util_threshold)
    return r


def b200_profile(hbm_gbs: float, bf16_tflops: float, decode_factor: float = 1.0) -> HardwareProfile:
    """The B200 the bench runs on, from MEASURED_PEAKS.json: beta = peak_mem_bw
    = measured copy bandwidth; gamma = the same (the decode of a stored element
    is fused into the HBM-bound attention read); peak_compute = bf16 dense."""
    bw = hbm_gbs * 1e9
    return HardwareProfile(hbm_bandwidth=bw, core_throughput=bw, decode_factor=decode_factor,
                           peak_compute=bf16_tflops * 1e12, peak_mem_bw=bw)
