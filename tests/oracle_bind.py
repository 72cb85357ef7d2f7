# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE — ctypes bindings of the CPU checkers.

``OracleEngine`` drives oracle/libpikv_oracle.so (our C restatement);
``RefEngine`` drives oracle/_ref/libpikv_ref.so (the reference's own objects,
built only where /root/reference exists).  Both expose the same per-stream
step() so tests can compare them with each other and with the GPU engine.
"""
from __future__ import annotations

import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import build as obuild  # noqa: E402
from paper_2508_06526_b200.config import EngineConfig, PikvConfigC  # noqa: E402
from paper_2508_06526_b200.wire import SNAPSHOT_DTYPE  # noqa: E402

c_double_p = ctypes.POINTER(ctypes.c_double)
c_u64_p = ctypes.POINTER(ctypes.c_uint64)
c_i64_p = ctypes.POINTER(ctypes.c_int64)
c_i32_p = ctypes.POINTER(ctypes.c_int32)


class PoEvict(ctypes.Structure):
    _fields_ = [("step", ctypes.c_uint64), ("id", ctypes.c_uint64), ("token", ctypes.c_int64),
                ("expert", ctypes.c_int32), ("device", ctypes.c_int32),
                ("score", ctypes.c_double), ("reason", ctypes.c_int32),
                ("stream", ctypes.c_int32)]


class PoStepOut(ctypes.Structure):
    _fields_ = [("experts", ctypes.c_int32 * 64), ("gates", ctypes.c_double * 64),
                ("logits", c_double_p),
                ("inserts", ctypes.c_int32), ("hits", ctypes.c_int32),
                ("lookups", ctypes.c_int32), ("n_attended", ctypes.c_int32),
                ("fetch_elements", ctypes.c_int64),
                ("pages_before", ctypes.c_int32), ("pages_after", ctypes.c_int32),
                ("evictions", ctypes.POINTER(PoEvict)), ("evict_cap", ctypes.c_int32),
                ("n_evictions", ctypes.c_int32),
                ("att_token", c_i64_p), ("att_expert", c_i32_p), ("att_weight", c_double_p),
                ("att_cap", ctypes.c_int32), ("y", c_double_p)]


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


_ORACLE = None
_REF = None


def oracle_lib():
    global _ORACLE
    if _ORACLE is None:
        lib = ctypes.CDLL(obuild.build_oracle())
        lib.po_engine_create.restype = ctypes.c_void_p
        lib.po_engine_create.argtypes = [ctypes.POINTER(PikvConfigC), c_double_p, c_double_p,
                                         c_double_p, c_i32_p, ctypes.POINTER(ctypes.c_int)]
        lib.po_engine_destroy.argtypes = [ctypes.c_void_p]
        lib.po_engine_step.argtypes = [ctypes.c_void_p, c_double_p, c_double_p, c_double_p,
                                       c_double_p, ctypes.POINTER(PoStepOut)]
        lib.po_engine_step_noattend.argtypes = lib.po_engine_step.argtypes
        lib.po_engine_slot_count.restype = ctypes.c_int64
        lib.po_engine_slot_count.argtypes = [ctypes.c_void_p]
        lib.po_engine_dump_slots.argtypes = [ctypes.c_void_p, c_u64_p, c_u64_p, c_i64_p, c_i32_p,
                                             c_u64_p, c_u64_p, c_u64_p, c_double_p, c_double_p]
        lib.po_engine_set_attn_mass.argtypes = [ctypes.c_void_p, c_double_p, c_double_p]
        lib.po_engine_read_payload.argtypes = [ctypes.c_void_p, ctypes.c_int64,
                                               ctypes.POINTER(ctypes.c_float),
                                               ctypes.POINTER(ctypes.c_float)]
        lib.po_engine_write_payload.argtypes = lib.po_engine_read_payload.argtypes
        lib.po_engine_step_embed.argtypes = [ctypes.c_void_p, c_double_p, c_double_p,
                                             ctypes.POINTER(PoStepOut), ctypes.c_int]
        lib.po_encoder_weights.argtypes = [ctypes.c_int, ctypes.c_uint64, c_double_p]
        lib.po_encode.argtypes = [c_double_p, ctypes.c_int, c_double_p, c_double_p, c_double_p,
                                  c_double_p]
        lib.po_engine_insert_bulk.argtypes = [ctypes.c_void_p, ctypes.c_int64, c_double_p,
                                              c_double_p, c_i32_p, c_double_p, c_i64_p]
        lib.po_engine_snapshot.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                           ctypes.c_int64, c_i64_p]
        lib.po_engine_router.restype = ctypes.c_void_p
        lib.po_engine_router.argtypes = [ctypes.c_void_p]
        lib.po_router_state.argtypes = [ctypes.c_void_p, c_double_p, c_u64_p, c_u64_p,
                                        c_double_p, c_u64_p, c_u64_p]
        lib.po_engine_sched_state.argtypes = [ctypes.c_void_p, c_double_p, c_double_p, c_u64_p]
        lib.po_engine_store_stats.argtypes = [ctypes.c_void_p, c_u64_p, c_u64_p, c_u64_p, c_u64_p]
        lib.po_engine_shards_per_device.argtypes = [ctypes.c_void_p]
        lib.po_engine_stored_width.argtypes = [ctypes.c_void_p]
        lib.po_normal_vector.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_double,
                                         c_double_p]
        lib.po_shard_assign.argtypes = [ctypes.c_int64] + [ctypes.c_int] * 5 + [
            ctypes.POINTER(ctypes.c_int)] * 3
        lib.po_select_evictions.argtypes = [c_double_p, c_u64_p, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_double,
                                            ctypes.POINTER(ctypes.c_int),
                                            ctypes.POINTER(ctypes.c_int)]
        lib.po_attention.argtypes = [c_double_p, c_double_p, c_double_p, ctypes.c_int,
                                     ctypes.c_int, c_double_p, c_double_p]
        lib.po_softmax.argtypes = [c_double_p, ctypes.c_int, c_double_p]
        lib.po_quantize_row.argtypes = [ctypes.POINTER(ctypes.c_float), ctypes.c_int,
                                        ctypes.c_int, ctypes.POINTER(ctypes.c_uint8),
                                        ctypes.POINTER(ctypes.c_float)]
        lib.po_dequantize_row.argtypes = [ctypes.POINTER(ctypes.c_uint8), ctypes.c_float,
                                          ctypes.c_int, ctypes.c_int,
                                          ctypes.POINTER(ctypes.c_float)]
        lib.po_router_create.restype = ctypes.c_void_p
        lib.po_router_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64]
        lib.po_router_destroy.argtypes = [ctypes.c_void_p]
        lib.po_route_logits.argtypes = [ctypes.c_void_p, ctypes.POINTER(PikvConfigC), c_double_p,
                                        ctypes.POINTER(ctypes.c_int), c_double_p]
        lib.po_route.argtypes = [ctypes.c_void_p, ctypes.POINTER(PikvConfigC), c_double_p,
                                 c_double_p, ctypes.POINTER(ctypes.c_int), c_double_p]
        lib.po_record_miss.argtypes = [ctypes.c_void_p, ctypes.c_int]
        lib.po_adapt.argtypes = [ctypes.c_void_p, ctypes.POINTER(PikvConfigC),
                                 ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_double]
        lib.po_router_set_state.argtypes = [ctypes.c_void_p, c_double_p, c_u64_p, c_u64_p,
                                            c_double_p, ctypes.c_uint64, ctypes.c_uint64]
        _ORACLE = lib
    return _ORACLE


def ref_lib():
    """The reference's own objects, or None when they cannot be built here."""
    global _REF
    if _REF is None:
        path = obuild.build_ref()
        if path is None or not os.path.exists(path):
            return None
        lib = ctypes.CDLL(path)
        lib.ref_create.restype = ctypes.c_void_p
        lib.ref_create.argtypes = [ctypes.POINTER(PikvConfigC), c_double_p,
                                   ctypes.POINTER(ctypes.c_int)]
        lib.ref_destroy.argtypes = [ctypes.c_void_p]
        lib.ref_step.argtypes = [ctypes.c_void_p, c_double_p, c_double_p, c_double_p, c_double_p,
                                 ctypes.POINTER(PoStepOut)]
        lib.ref_step_noattend.argtypes = lib.ref_step.argtypes
        lib.ref_dump_slots.argtypes = [ctypes.c_void_p, c_u64_p, c_u64_p, c_i64_p, c_i32_p,
                                       c_u64_p, c_u64_p, c_u64_p, c_double_p]
        lib.ref_snapshot.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                     ctypes.c_int64, c_i64_p]
        lib.ref_router_state.argtypes = [ctypes.c_void_p, c_double_p, c_u64_p, c_u64_p,
                                         c_double_p, c_u64_p, c_u64_p]
        lib.ref_sched_state.argtypes = [ctypes.c_void_p, c_double_p, c_double_p, c_u64_p]
        lib.ref_shards_per_device.argtypes = [ctypes.c_void_p]
        lib.ref_shard_assign.argtypes = lib_shard_argtypes()
        lib.ref_select_evictions.argtypes = [c_double_p, c_u64_p, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int, ctypes.c_double,
                                             ctypes.POINTER(ctypes.c_int),
                                             ctypes.POINTER(ctypes.c_int)]
        lib.ref_attention.argtypes = [c_double_p, c_double_p, c_double_p, ctypes.c_int,
                                      ctypes.c_int, c_double_p, c_double_p]
        lib.ref_time_streams.restype = ctypes.c_double
        lib.ref_time_streams.argtypes = [ctypes.POINTER(PikvConfigC), ctypes.c_int, ctypes.c_long,
                                         ctypes.c_int, ctypes.c_uint64, c_double_p,
                                         ctypes.POINTER(ctypes.c_long)]
        _REF = lib
    return _REF


def lib_shard_argtypes():
    return [ctypes.c_int64] + [ctypes.c_int] * 5 + [ctypes.POINTER(ctypes.c_int)] * 3


def normal_vector(seed: int, n: int, scale: float = 1.0) -> np.ndarray:
    """pikv::Rng(seed).normal_vector(n, scale) (rng.hpp:54-58), bit-exact."""
    out = np.empty(n, dtype=np.float64)
    oracle_lib().po_normal_vector(seed, n, scale, _ptr(out, c_double_p))
    return out


def round_to(x: np.ndarray, dtype: str) -> np.ndarray:
    """Round to the storage dtype (RNE) and return float64."""
    x = np.asarray(x, dtype=np.float64)
    if dtype == "f32":
        return x.astype(np.float32).astype(np.float64)
    f = x.astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    finite = (u & 0x7F800000) != 0x7F800000
    u = np.where(finite, u + 0x7FFF + ((u >> 16) & 1), u) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


class _StepMixin:
    E: int
    k: int
    dp: int

    def _new_out(self, evict_cap=4096, att_cap=1 << 16):
        out = PoStepOut()
        self._logits = np.zeros(self.E, dtype=np.float64)
        self._ev = (PoEvict * evict_cap)()
        self._att_t = np.zeros(att_cap, dtype=np.int64)
        self._att_e = np.zeros(att_cap, dtype=np.int32)
        self._att_w = np.zeros(att_cap, dtype=np.float64)
        self._y = np.zeros(self.dp, dtype=np.float64)
        out.logits = _ptr(self._logits, c_double_p)
        out.evictions = self._ev
        out.evict_cap = evict_cap
        out.att_token = _ptr(self._att_t, c_i64_p)
        out.att_expert = _ptr(self._att_e, c_i32_p)
        out.att_weight = _ptr(self._att_w, c_double_p)
        out.att_cap = att_cap
        out.y = _ptr(self._y, c_double_p)
        return out

    def _collect(self, out):
        n_att = min(out.n_attended, out.att_cap)
        nev = min(out.n_evictions, out.evict_cap)
        evs = [(int(e.step), int(e.id), int(e.token), int(e.expert), int(e.device),
                float(e.score), int(e.reason)) for e in self._ev[:nev]]
        return {
            "experts": [out.experts[j] for j in range(self.k)],
            "gates": np.array([out.gates[j] for j in range(self.k)]),
            "logits": self._logits.copy(),
            "inserts": out.inserts, "hits": out.hits, "lookups": out.lookups,
            "n_attended": out.n_attended, "fetch_elements": out.fetch_elements,
            "pages_before": out.pages_before, "pages_after": out.pages_after,
            "evictions": evs,
            "att_token": self._att_t[:n_att].copy(), "att_expert": self._att_e[:n_att].copy(),
            "att_weight": self._att_w[:n_att].copy(),
            "y": self._y.copy(),
        }


class OracleEngine(_StepMixin):
    """One decode stream of the C restatement (pikv_oracle.c)."""

    def __init__(self, cfg: EngineConfig, w_r=None, basis=None, bias=None, kept=None,
                 evict_cap=4096, att_cap=1 << 16):
        self.lib = oracle_lib()
        self.cfg = cfg
        self.E, self.k, self.dp = cfg.model.E, cfg.router.k, cfg.stored_width
        self._c = cfg.to_c()
        err = ctypes.c_int(0)
        arrs = [None if a is None else np.ascontiguousarray(a, dtype=np.float64)
                for a in (w_r, basis, bias)]
        kp = None if kept is None else np.ascontiguousarray(kept, dtype=np.int32)
        self._keep = arrs + [kp]
        self.h = self.lib.po_engine_create(ctypes.byref(self._c), _ptr(arrs[0], c_double_p),
                                           _ptr(arrs[1], c_double_p), _ptr(arrs[2], c_double_p),
                                           _ptr(kp, c_i32_p), ctypes.byref(err))
        if not self.h:
            raise RuntimeError("po_engine_create failed: %d" % err.value)
        self.error = err.value
        self.out = self._new_out(evict_cap, att_cap)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.po_engine_destroy(self.h)
            self.h = None

    def step(self, q, k, v, saliency=None, attend=True):
        q, k, v = (np.ascontiguousarray(a, dtype=np.float64) for a in (q, k, v))
        sal = None if saliency is None else np.ascontiguousarray(saliency, dtype=np.float64)
        fn = self.lib.po_engine_step if attend else self.lib.po_engine_step_noattend
        rc = fn(self.h, _ptr(q, c_double_p), _ptr(k, c_double_p), _ptr(v, c_double_p),
                _ptr(sal, c_double_p), ctypes.byref(self.out))
        if rc:
            raise RuntimeError("oracle step error %d" % rc)
        return self._collect(self.out)

    def slots(self):
        n = self.lib.po_engine_slot_count(self.h)
        cols = {"id": np.uint64, "shard_seq": np.uint64, "token": np.int64, "expert": np.int32,
                "insert_step": np.uint64, "last_access": np.uint64, "freq": np.uint64,
                "attn_mass": np.float64}
        out = {k: np.zeros(n, dtype=t) for k, t in cols.items()}
        nl = max(self.cfg.n_layers, 0)
        out["per_layer"] = np.zeros(n * max(nl, 1), dtype=np.float64)
        self.lib.po_engine_dump_slots(
            self.h, _ptr(out["id"], c_u64_p), _ptr(out["shard_seq"], c_u64_p),
            _ptr(out["token"], c_i64_p), _ptr(out["expert"], c_i32_p),
            _ptr(out["insert_step"], c_u64_p), _ptr(out["last_access"], c_u64_p),
            _ptr(out["freq"], c_u64_p), _ptr(out["attn_mass"], c_double_p),
            _ptr(out["per_layer"], c_double_p))
        return out

    def step_embed(self, emb, saliency=None, attend=True):
        """Engine::step(TokenInput{embedding}) incl. the QueryEncoder."""
        x = np.ascontiguousarray(emb, dtype=np.float64)
        sal = None if saliency is None else np.ascontiguousarray(saliency, dtype=np.float64)
        rc = self.lib.po_engine_step_embed(self.h, _ptr(x, c_double_p), _ptr(sal, c_double_p),
                                           ctypes.byref(self.out), 1 if attend else 0)
        if rc:
            raise RuntimeError("oracle step error %d" % rc)
        return self._collect(self.out)

    def insert_bulk(self, k, v, experts, saliency=None) -> int:
        """The store build of a prefill restated (po_engine_insert_bulk)."""
        k, v = (np.ascontiguousarray(a, dtype=np.float64) for a in (k, v))
        ex = np.ascontiguousarray(experts, dtype=np.int32)
        sal = None if saliency is None else np.ascontiguousarray(saliency, dtype=np.float64)
        nd = ctypes.c_int64(0)
        rc = self.lib.po_engine_insert_bulk(self.h, ex.shape[0], _ptr(k, c_double_p),
                                            _ptr(v, c_double_p), _ptr(ex, c_i32_p),
                                            _ptr(sal, c_double_p), ctypes.byref(nd))
        if rc:
            raise RuntimeError("oracle insert_bulk error %d" % rc)
        return nd.value

    def snapshot(self, now):
        """KVStore::snapshot(now) restated (po_engine_snapshot)."""
        n = ctypes.c_int64(0)
        self.lib.po_engine_snapshot(self.h, now, None, 0, ctypes.byref(n))
        out = np.zeros(n.value, dtype=SNAPSHOT_DTYPE)
        self.lib.po_engine_snapshot(self.h, now, out.ctypes.data, n.value, ctypes.byref(n))
        return out

    def read_payload(self, slots):
        """Stored K, V (as attended) of the given slots, [n][d'] float32."""
        fp = ctypes.POINTER(ctypes.c_float)
        k = np.zeros((len(slots), self.dp), dtype=np.float32)
        v = np.zeros((len(slots), self.dp), dtype=np.float32)
        for i, gi in enumerate(slots):
            self.lib.po_engine_read_payload(self.h, int(gi), k[i].ctypes.data_as(fp),
                                            v[i].ctypes.data_as(fp))
        return k, v

    def write_payload(self, slots, k, v):
        """Overwrite the stored K/V of live slots ([n][d'] float32 each)."""
        fp = ctypes.POINTER(ctypes.c_float)
        k = np.ascontiguousarray(k, dtype=np.float32)
        v = np.ascontiguousarray(v, dtype=np.float32)
        for i, gi in enumerate(slots):
            rc = self.lib.po_engine_write_payload(self.h, int(gi), k[i].ctypes.data_as(fp),
                                                  v[i].ctypes.data_as(fp))
            if rc:
                raise RuntimeError("write_payload: slot %d not live" % gi)

    def set_attn_mass(self, attn_mass, per_layer=None):
        a = np.ascontiguousarray(attn_mass, dtype=np.float64)
        p = None if per_layer is None else np.ascontiguousarray(per_layer, dtype=np.float64)
        self.lib.po_engine_set_attn_mass(self.h, _ptr(a, c_double_p), _ptr(p, c_double_p))

    def router_state(self):
        E = self.E
        load = np.zeros(E)
        usage = np.zeros(E, dtype=np.uint64)
        miss = np.zeros(E, dtype=np.uint64)
        bias = np.zeros(E)
        step = ctypes.c_uint64(0)
        tot = ctypes.c_uint64(0)
        self.lib.po_router_state(self.lib.po_engine_router(self.h), _ptr(load, c_double_p),
                                 _ptr(usage, c_u64_p), _ptr(miss, c_u64_p),
                                 _ptr(bias, c_double_p), ctypes.byref(step), ctypes.byref(tot))
        return {"load": load, "usage": usage, "miss": miss, "bias": bias, "step": step.value,
                "total_usage": tot.value}

    def sched_state(self):
        th, rh, st = ctypes.c_double(), ctypes.c_double(), ctypes.c_uint64()
        self.lib.po_engine_sched_state(self.h, ctypes.byref(th), ctypes.byref(rh),
                                       ctypes.byref(st))
        return {"theta": th.value, "running_hit": rh.value, "step": st.value}

    def store_stats(self):
        vals = [ctypes.c_uint64() for _ in range(4)]
        self.lib.po_engine_store_stats(self.h, *[ctypes.byref(v) for v in vals])
        return dict(zip(("live", "memory_bytes", "inserts", "overwrites"),
                        [v.value for v in vals]))


class RefEngine(_StepMixin):
    """One decode stream driven through the reference's own objects."""

    def __init__(self, cfg: EngineConfig, w_r=None):
        self.lib = ref_lib()
        if self.lib is None:
            raise RuntimeError("reference objects unavailable")
        self.cfg = cfg
        self.E, self.k, self.dp = cfg.model.E, cfg.router.k, cfg.stored_width
        self._c = cfg.to_c()
        err = ctypes.c_int(0)
        self._w = None if w_r is None else np.ascontiguousarray(w_r, dtype=np.float64)
        self.h = self.lib.ref_create(ctypes.byref(self._c), _ptr(self._w, c_double_p),
                                     ctypes.byref(err))
        if not self.h:
            raise RuntimeError("ref_create failed: %d" % err.value)
        self.out = self._new_out()

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_destroy(self.h)
            self.h = None

    def step(self, q, k, v, saliency=None, attend=True):
        q, k, v = (np.ascontiguousarray(a, dtype=np.float64) for a in (q, k, v))
        sal = None if saliency is None else np.ascontiguousarray(saliency, dtype=np.float64)
        fn = self.lib.ref_step if attend else self.lib.ref_step_noattend
        rc = fn(self.h, _ptr(q, c_double_p), _ptr(k, c_double_p), _ptr(v, c_double_p),
                _ptr(sal, c_double_p), ctypes.byref(self.out))
        if rc:
            raise RuntimeError("ref step error %d" % rc)
        return self._collect(self.out)

    def snapshot(self, now):
        """The reference's own KVStore::snapshot(now)."""
        n = ctypes.c_int64(0)
        self.lib.ref_snapshot(self.h, now, None, 0, ctypes.byref(n))
        out = np.zeros(n.value, dtype=SNAPSHOT_DTYPE)
        self.lib.ref_snapshot(self.h, now, out.ctypes.data, n.value, ctypes.byref(n))
        return out

    def slots(self, n_slots):
        cols = {"id": np.uint64, "shard_seq": np.uint64, "token": np.int64, "expert": np.int32,
                "insert_step": np.uint64, "last_access": np.uint64, "freq": np.uint64,
                "attn_mass": np.float64}
        out = {k: np.zeros(n_slots, dtype=t) for k, t in cols.items()}
        self.lib.ref_dump_slots(
            self.h, _ptr(out["id"], c_u64_p), _ptr(out["shard_seq"], c_u64_p),
            _ptr(out["token"], c_i64_p), _ptr(out["expert"], c_i32_p),
            _ptr(out["insert_step"], c_u64_p), _ptr(out["last_access"], c_u64_p),
            _ptr(out["freq"], c_u64_p), _ptr(out["attn_mass"], c_double_p))
        return out

    def router_state(self):
        E = self.E
        load = np.zeros(E)
        usage = np.zeros(E, dtype=np.uint64)
        miss = np.zeros(E, dtype=np.uint64)
        bias = np.zeros(E)
        step = ctypes.c_uint64(0)
        tot = ctypes.c_uint64(0)
        self.lib.ref_router_state(self.h, _ptr(load, c_double_p), _ptr(usage, c_u64_p),
                                  _ptr(miss, c_u64_p), _ptr(bias, c_double_p),
                                  ctypes.byref(step), ctypes.byref(tot))
        return {"load": load, "usage": usage, "miss": miss, "bias": bias, "step": step.value,
                "total_usage": tot.value}

    def sched_state(self):
        th, rh, st = ctypes.c_double(), ctypes.c_double(), ctypes.c_uint64()
        self.lib.ref_sched_state(self.h, ctypes.byref(th), ctypes.byref(rh), ctypes.byref(st))
        return {"theta": th.value, "running_hit": rh.value, "step": st.value}


def make_stream(T: int, d: int, seed: int, dtype: str = "f32", n_layers: int = 0):
    """Synthetic (q, k, v, saliency) per token: pikv::Rng(seed) N(0,1) rounded to dtype."""
    raw = normal_vector(seed, T * (3 * d + n_layers))
    raw = raw.reshape(T, 3 * d + n_layers)
    q = round_to(raw[:, :d], dtype)
    k = round_to(raw[:, d:2 * d], dtype)
    v = round_to(raw[:, 2 * d:3 * d], dtype)
    sal = np.abs(raw[:, 3 * d:]) * 0.1 if n_layers else None
    return q, k, v, sal


def oracle_encode(width: int, seed: int, x):
    """QueryEncoder restated (po_encoder_weights + po_encode)."""
    lib = oracle_lib()
    w = np.zeros(3 * width * width)
    lib.po_encoder_weights(width, seed, _ptr(w, c_double_p))
    x = np.ascontiguousarray(x, dtype=np.float64)
    q, k, v = (np.zeros(width) for _ in range(3))
    lib.po_encode(_ptr(w, c_double_p), width, _ptr(x, c_double_p), _ptr(q, c_double_p),
                  _ptr(k, c_double_p), _ptr(v, c_double_p))
    return q, k, v
