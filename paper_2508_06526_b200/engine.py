# SPDX-License-Identifier: Apache-2.0
"""Python mirror of the reference's decode-path API over the C-ABI.

Names and argument meanings follow /root/reference/proj/include/pikv:
``shard_assign`` (kvstore.hpp:25-26), ``select_evictions`` (scheduler.hpp:
114-116), ``attention`` (pipeline.hpp:46-47), ``Engine.step`` (pipeline.hpp:
105) with ``store()``/``router_state()``/``scheduler_state()`` views.  Errors
raise ``PikvError`` whose ``kind`` is the reference exception class name.
Every compute call runs on the GPU through libpikv_b200.so; torch is used only
to own device buffers.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _capi
from ._capi import PikvError, PikvEvictRecord, PikvStepSummary, check, lib
from .config import REASON, EngineConfig

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None


def _dev(a, dtype) -> "torch.Tensor":
    t = torch.as_tensor(np.ascontiguousarray(a, dtype=dtype))
    return t.cuda()


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _np_ptr(a) -> Optional[int]:
    return None if a is None else a.ctypes.data


# ---------------------------------------------------------------------------
# free functions
# ---------------------------------------------------------------------------
@dataclass
class ShardId:  # kvstore.hpp:14-20
    device: int
    shard_index: int
    raw: int


def shard_assign(t, e, n_tok: int, n_exp: int, devices: int, additive: bool = False):
    """kvstore.cpp:14-30.  Scalars -> ShardId; arrays -> (device, shard, raw) arrays."""
    scalar = np.isscalar(t) and np.isscalar(e)
    tt = np.atleast_1d(np.asarray(t, dtype=np.int64))
    ee = np.atleast_1d(np.asarray(e, dtype=np.int32))
    n = int(tt.size)
    td, ed = _dev(tt, np.int64), _dev(ee, np.int32)
    dev = torch.empty(n, dtype=torch.int32, device="cuda")
    sh = torch.empty_like(dev)
    raw = torch.empty_like(dev)
    check(lib().pikv_shard_assign(_ptr(td), _ptr(ed), n, n_tok, n_exp, devices, int(additive),
                                  _ptr(dev), _ptr(sh), _ptr(raw)))
    d_, s_, r_ = dev.cpu().numpy(), sh.cpu().numpy(), raw.cpu().numpy()
    if scalar:
        return ShardId(int(d_[0]), int(s_[0]), int(r_[0]))
    return d_, s_, r_


def select_evictions(pages: Sequence[Tuple[float, int]], budget_pages: int, use_theta: bool,
                     theta: float) -> List[Tuple[int, str]]:
    """scheduler.cpp:231-260: [(page index, reason)] in eviction order."""
    n = len(pages)
    agg = _dev([p[0] for p in pages] or [0.0], np.float64)
    old = _dev([p[1] for p in pages] or [0], np.uint64)
    idx = torch.zeros(max(n, 1), dtype=torch.int32, device="cuda")
    why = torch.zeros_like(idx)
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    check(lib().pikv_select_evictions(_ptr(agg), _ptr(old), n, budget_pages, int(use_theta),
                                      float(theta), _ptr(idx), _ptr(why), _ptr(cnt)))
    m = int(cnt.item())
    return [(int(i), REASON[int(r)]) for i, r in zip(idx.cpu().numpy()[:m], why.cpu().numpy()[:m])]


def attention(query, keys, values):
    """pipeline.cpp:59-85 on the GPU (fp32): returns (output, weights)."""
    q = np.asarray(query, dtype=np.float32).reshape(1, -1)
    w = q.shape[1]
    k = np.asarray(keys, dtype=np.float32).reshape(-1, w)
    v = np.asarray(values, dtype=np.float32).reshape(-1, w)
    n = k.shape[0]
    if n == 0:
        return np.zeros(w, dtype=np.float32), np.zeros(0, dtype=np.float32)
    qd, kd, vd = _dev(q, np.float32), _dev(k, np.float32), _dev(v, np.float32)
    y = torch.empty(w, dtype=torch.float32, device="cuda")
    wt = torch.empty(n, dtype=torch.float32, device="cuda")
    check(lib().pikv_attention(_ptr(qd), _ptr(kd), _ptr(vd), 1, n, w, _ptr(y), _ptr(wt)))
    return y.cpu().numpy(), wt.cpu().numpy()


def quantize(x, bits: int):
    """This engine's symmetric absmax int8/int4 quantizer: (codes, scales) per row."""
    x = np.asarray(x, dtype=np.float32)
    rows, width = x.shape
    xd = _dev(x, np.float32)
    codes = torch.empty(rows * (width if bits == 8 else width // 2), dtype=torch.uint8,
                        device="cuda")
    scales = torch.empty(rows, dtype=torch.float32, device="cuda")
    check(lib().pikv_quantize(_ptr(xd), 0, rows, width, bits, _ptr(codes), _ptr(scales)))
    return codes.cpu().numpy().reshape(rows, -1), scales.cpu().numpy()


def dequantize(codes, scales, width: int, bits: int):
    codes = np.asarray(codes, dtype=np.uint8)
    rows = codes.shape[0]
    cd, sd = _dev(codes, np.uint8), _dev(scales, np.float32)
    out = torch.empty(rows * width, dtype=torch.float32, device="cuda")
    check(lib().pikv_dequantize(_ptr(cd), _ptr(sd), rows, width, bits, _ptr(out)))
    return out.cpu().numpy().reshape(rows, width)


def lowrank_encode(x, basis, bias=None):
    """project_encode per head (compressor.cpp:318-329): x [rows][H*hd] -> [rows][H*r]."""
    basis = np.asarray(basis, dtype=np.float32)
    H, r, hd = basis.shape
    x = np.asarray(x, dtype=np.float32).reshape(-1, H * hd)
    rows = x.shape[0]
    y = torch.empty(rows * H * r, dtype=torch.float32, device="cuda")
    b = None if bias is None else _dev(bias, np.float32)
    xd, bd = _dev(x, np.float32), _dev(basis, np.float32)
    check(lib().pikv_lowrank_encode(_ptr(xd), _ptr(bd), _ptr(b), rows, H, hd, r, _ptr(y)))
    return y.cpu().numpy().reshape(rows, H * r)


def lowrank_decode(y, basis, bias=None):
    """project_decode per head (compressor.cpp:331-340)."""
    basis = np.asarray(basis, dtype=np.float32)
    H, r, hd = basis.shape
    y = np.asarray(y, dtype=np.float32).reshape(-1, H * r)
    rows = y.shape[0]
    x = torch.empty(rows * H * hd, dtype=torch.float32, device="cuda")
    b = None if bias is None else _dev(bias, np.float32)
    yd, bd = _dev(y, np.float32), _dev(basis, np.float32)
    check(lib().pikv_lowrank_decode(_ptr(yd), _ptr(bd), _ptr(b), rows, H, hd, r, _ptr(x)))
    return x.cpu().numpy().reshape(rows, H * hd)


# ---------------------------------------------------------------------------
# engine
# ---------------------------------------------------------------------------
@dataclass
class EvictionRecord:  # scheduler.hpp:90-98
    step: int
    entry_id: int
    token_id: int
    expert_id: int
    device: int
    score: float
    reason: str
    stream: int = 0


class Engine:
    """B streams of ``pikv::Engine`` (pipeline.hpp:101-145) on one GPU."""

    def __init__(self, cfg: EngineConfig, device: int = 0):
        self.cfg = cfg
        self._c = cfg.to_c()
        h = ctypes.c_void_p()
        check(lib().pikv_engine_create(ctypes.byref(self._c), device, ctypes.byref(h)))
        self.h = h
        self.device = device
        self.B = cfg.batch
        self.E, self.k = cfg.model.E, cfg.router.k
        self.dp = cfg.stored_width
        self.d = cfg.model.d

    @classmethod
    def _borrowed(cls, cfg: EngineConfig, handle, device: int):
        """An engine owned by a group (not destroyed by this object)."""
        self = cls.__new__(cls)
        self.cfg, self._c = cfg, cfg.to_c()
        self.h, self._owned, self.device = ctypes.c_void_p(handle), False, device
        self.B = cfg.batch
        self.E, self.k = cfg.model.E, cfg.router.k
        self.dp = cfg.stored_width
        self.d = cfg.model.d
        return self

    def close(self):
        h, self.h = getattr(self, "h", None), None
        if h and getattr(self, "_owned", True):
            try:
                lib().pikv_engine_destroy(h)
            except (AttributeError, TypeError):  # interpreter shutdown: modules torn down
                pass

    __del__ = close

    # ---- configuration --------------------------------------------------
    def set_router_matrix(self, w_r):
        w = np.ascontiguousarray(w_r, dtype=np.float64)
        check(lib().pikv_set_router_matrix_host(self.h, _np_ptr(w)))

    def set_codec(self, basis=None, bias=None, kept=None):
        b = None if basis is None else np.ascontiguousarray(basis, dtype=np.float32)
        c = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
        k = None if kept is None else np.ascontiguousarray(kept, dtype=np.int32)
        self._codec_keep = (b, c, k)
        check(lib().pikv_set_codec_host(self.h, _np_ptr(b), _np_ptr(c), _np_ptr(k)))

    # ---- stepping ---------------------------------------------------------
    def step(self, q, k, v, saliency=None, y=None):
        """Engine::step for all streams on device tensors [B][d] (kv dtype)."""
        if y is None:
            y = torch.empty(self.B, self.dp, dtype=torch.float32, device="cuda")
        es = self.external_stream()
        es.wait_stream(torch.cuda.current_stream())
        check(lib().pikv_step(self.h, _ptr(q), _ptr(k), _ptr(v), _ptr(saliency), _ptr(y)))
        torch.cuda.current_stream().wait_stream(es)
        return y

    def external_stream(self):
        """The engine's CUDA stream as a torch stream object (ordering only)."""
        if getattr(self, "_ext", None) is None:
            self._ext = torch.cuda.ExternalStream(self.stream_handle())
        return self._ext

    def step_host(self, q, k, v, saliency=None):
        """Engine::step through host buffers (numpy); returns y [B][d'] fp32."""
        dt = np.float32 if self.cfg.kv_dtype == "f32" else np.uint16
        q, k, v = (np.ascontiguousarray(a).view(dt) if a.dtype != dt else
                   np.ascontiguousarray(a) for a in (q, k, v))
        sal = None if saliency is None else np.ascontiguousarray(saliency, dtype=np.float64)
        y = np.empty((self.B, self.dp), dtype=np.float32)
        check(lib().pikv_step_host(self.h, _np_ptr(q), _np_ptr(k), _np_ptr(v), _np_ptr(sal),
                                   _np_ptr(y)))
        return y

    def step_embed(self, emb, saliency=None, y=None):
        """Engine::step(TokenInput{embedding}) for all streams: device fp64
        tensor [B][d]; the QueryEncoder runs on the GPU (pipeline.cpp:222)."""
        if y is None:
            y = torch.empty(self.B, self.dp, dtype=torch.float32, device="cuda")
        es = self.external_stream()
        es.wait_stream(torch.cuda.current_stream())
        check(lib().pikv_step_embed(self.h, _ptr(emb), _ptr(saliency), _ptr(y)))
        torch.cuda.current_stream().wait_stream(es)
        return y

    def step_embed_host(self, emb, saliency=None):
        """Engine::step(TokenInput{embedding}) through host buffers (numpy
        fp64 [B][d]); returns y [B][d'] fp32."""
        x = np.ascontiguousarray(emb, dtype=np.float64)
        sal = None if saliency is None else np.ascontiguousarray(saliency, dtype=np.float64)
        y = np.empty((self.B, self.dp), dtype=np.float32)
        check(lib().pikv_step_embed_host(self.h, _np_ptr(x), _np_ptr(sal), _np_ptr(y)))
        return y

    def insert_bulk_host(self, stream: int, k, v, experts, saliency=None) -> int:
        """The store build of a prefill (pikv_insert_bulk_host): T tokens with
        given experts [T][k]; k/v [T][d] numpy in the engine's kv dtype
        (uint16 bf16 bits or float32).  Returns the displacement count."""
        dt = np.float32 if self.cfg.kv_dtype == "f32" else np.uint16
        k, v = (np.ascontiguousarray(a).view(dt) if a.dtype != dt else np.ascontiguousarray(a)
                for a in (k, v))
        ex = np.ascontiguousarray(experts, dtype=np.int32)
        sal = None if saliency is None else np.ascontiguousarray(saliency, dtype=np.float64)
        nd = ctypes.c_int64(0)
        check(lib().pikv_insert_bulk_host(self.h, stream, int(ex.shape[0]), _np_ptr(k), _np_ptr(v),
                                          _np_ptr(ex), _np_ptr(sal), ctypes.byref(nd)))
        return nd.value

    def set_encoder(self, w_query, w_key, w_value):
        """Replace the seeded QueryEncoder's [d][d] matrices."""
        ws = [np.ascontiguousarray(w, dtype=np.float64) for w in (w_query, w_key, w_value)]
        check(lib().pikv_set_encoder_host(self.h, *[_np_ptr(w) for w in ws]))

    def prefill_synthetic(self, tokens: int, seed: int = 1):
        check(lib().pikv_prefill_synthetic(self.h, int(tokens), int(seed)))

    def fill_synthetic(self, q, k, v, seed: int):
        check(lib().pikv_fill_synthetic(self.h, _ptr(q), _ptr(k), _ptr(v), int(seed)))

    def sync(self):
        check(lib().pikv_sync(self.h))

    # ---- results ------------------------------------------------------------
    def read_step(self):
        B, k, E = self.B, self.k, self.E
        experts = np.zeros((B, k), dtype=np.int32)
        gates = np.zeros((B, k), dtype=np.float64)
        logits = np.zeros((B, E), dtype=np.float64)
        summ = (PikvStepSummary * B)()
        check(lib().pikv_read_step_host(self.h, _np_ptr(experts), _np_ptr(gates),
                                        _np_ptr(logits), ctypes.addressof(summ)))
        summary = [{f: getattr(s, f) for f, _ in PikvStepSummary._fields_} for s in summ]
        return experts, gates, logits, summary

    def read_evictions(self, cap: int = 1 << 20) -> List[EvictionRecord]:
        n = ctypes.c_int32(0)
        check(lib().pikv_read_evictions_host(self.h, None, 0, ctypes.byref(n)))  # count
        cap = min(cap, n.value)
        buf = (PikvEvictRecord * max(cap, 1))()
        check(lib().pikv_read_evictions_host(self.h, ctypes.addressof(buf), cap, ctypes.byref(n)))
        return [EvictionRecord(r.step, r.entry_id, r.token_id, r.expert_id, r.device, r.score,
                               REASON[r.reason], r.stream) for r in buf[:min(n.value, cap)]]

    def read_attended(self, stream: int, cap: int = 1 << 22):
        n = ctypes.c_int32(0)
        check(lib().pikv_read_attended_host(self.h, stream, None, None, None, 0, ctypes.byref(n)))
        m = n.value
        tok = np.zeros(max(m, 1), dtype=np.int64)
        ex = np.zeros(max(m, 1), dtype=np.int32)
        al = np.zeros(max(m, 1), dtype=np.float64)
        check(lib().pikv_read_attended_host(self.h, stream, _np_ptr(tok), _np_ptr(ex),
                                            _np_ptr(al), m, ctypes.byref(n)))
        return tok[:m], ex[:m], al[:m]

    def snapshot(self, stream: int, now: int = -1):
        """KVStore::snapshot(now) (kvstore.cpp:206-221) of `stream`, computed on
        the GPU: live entries of this rank's devices as a wire.SNAPSHOT_DTYPE
        array sorted by (device, shard, token, expert); now < 0 = the
        stream's current step.  wire.store_dump_lines() gives runner.cpp's
        JSONL."""
        from .wire import SNAPSHOT_DTYPE
        n = ctypes.c_int64(0)
        check(lib().pikv_snapshot_host(self.h, stream, now, None, 0, ctypes.byref(n)))
        out = np.zeros(n.value, dtype=SNAPSHOT_DTYPE)
        if n.value:
            check(lib().pikv_snapshot_host(self.h, stream, now, out.ctypes.data, n.value,
                                           ctypes.byref(n)))
        return out

    def slots(self, stream: int):
        n = lib().pikv_slot_count(self.h)
        cols = {"id": np.uint64, "shard_seq": np.uint64, "token": np.int64, "expert": np.int32,
                "insert_step": np.uint64, "last_access": np.uint64, "freq": np.uint64,
                "attn_mass": np.float64}
        out = {c: np.zeros(n, dtype=t) for c, t in cols.items()}
        nl = self.cfg.n_layers
        out["per_layer"] = np.zeros(n * max(nl, 1), dtype=np.float64)
        check(lib().pikv_read_slots_host(self.h, stream, *[_np_ptr(out[c]) for c in cols],
                                         _np_ptr(out["per_layer"]) if nl > 0 else None))
        return out

    def read_entries(self, stream: int, slots):
        """Stored K, V of stream-local slots decoded to fp32 ([n][d'] each)."""
        sl = np.ascontiguousarray(slots, dtype=np.int64)
        k = np.zeros((len(sl), self.dp), dtype=np.float32)
        v = np.zeros((len(sl), self.dp), dtype=np.float32)
        check(lib().pikv_read_entries_host(self.h, stream, _np_ptr(sl), len(sl), _np_ptr(k), _np_ptr(v)))
        return k, v

    def set_attn_mass(self, stream: int, attn_mass, per_layer=None):
        a = np.ascontiguousarray(attn_mass, dtype=np.float64)
        p = None if per_layer is None else np.ascontiguousarray(per_layer, dtype=np.float64)
        check(lib().pikv_write_attn_mass_host(self.h, stream, _np_ptr(a), _np_ptr(p)))

    def router_state(self, stream: int):
        E = self.E
        load = np.zeros(E)
        usage = np.zeros(E, dtype=np.uint64)
        miss = np.zeros(E, dtype=np.uint64)
        bias = np.zeros(E)
        step = np.zeros(1, dtype=np.uint64)
        tot = np.zeros(1, dtype=np.uint64)
        check(lib().pikv_read_router_state_host(self.h, stream, *[_np_ptr(a) for a in
                                                                  (load, usage, miss, bias,
                                                                   step, tot)]))
        return {"load": load, "usage": usage, "miss": miss, "bias": bias, "step": int(step[0]),
                "total_usage": int(tot[0])}

    def scheduler_state(self, stream: int):
        th = np.zeros(1)
        rh = np.zeros(1)
        st = np.zeros(1, dtype=np.uint64)
        check(lib().pikv_read_sched_state_host(self.h, stream, _np_ptr(th), _np_ptr(rh),
                                               _np_ptr(st)))
        return {"theta": float(th[0]), "running_hit": float(rh[0]), "step": int(st[0])}

    def store_stats(self, stream: int):
        vals = np.zeros(4, dtype=np.uint64)
        check(lib().pikv_store_stats_host(self.h, stream, *[_np_ptr(vals[i:i + 1])
                                                            for i in range(4)]))
        return dict(zip(("live", "memory_bytes", "inserts", "overwrites"), map(int, vals)))

    def pool_pages_in_use(self) -> int:
        return int(lib().pikv_pool_pages_in_use(self.h))

    def entry_bytes(self) -> int:
        return int(lib().pikv_entry_bytes(self.h))

    def kernel_launches(self) -> int:
        return int(lib().pikv_kernel_launches(self.h))

    def set_profiling(self, on: bool):
        check(lib().pikv_set_profiling(self.h, int(on)))

    PHASES = ("route", "insert", "sched_pages", "sched_select", "retr_count", "retr_scan",
              "retr_write", "attend", "combine", "finish_merge", "foldback", "feedback")

    def read_profile(self):
        """{phase: summed ms} over the steps run since set_profiling(True), and the count."""
        ms = np.zeros(len(self.PHASES), dtype=np.float32)
        n = ctypes.c_int32(0)
        check(lib().pikv_read_profile_host(self.h, _np_ptr(ms), len(self.PHASES),
                                           ctypes.byref(n)))
        return dict(zip(self.PHASES, ms.tolist())), int(n.value)

    # ---- multi-rank (see parallel.py) --------------------------------------
    def exchange_bytes(self) -> int:
        return int(lib().pikv_exchange_bytes(self.h))

    def step_local(self, q, k, v, saliency=None) -> int:
        ex = ctypes.c_void_p()
        check(lib().pikv_step_local(self.h, _ptr(q), _ptr(k), _ptr(v), _ptr(saliency),
                                    ctypes.byref(ex)))
        return ex.value

    def step_finish(self, gathered, y=None):
        if y is None:
            y = torch.empty(self.B, self.dp, dtype=torch.float32, device="cuda")
        check(lib().pikv_step_finish(self.h, _ptr(gathered), _ptr(y)))
        return y

    # ---- multi-GPU: NCCL inside the library --------------------------------
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        check(lib().pikv_nccl_unique_id(buf))
        return buf.raw

    def attach_nccl(self, uid: bytes):
        """ncclCommInitRank(world_size, uid, rank_id) -- collective over ranks."""
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        check(lib().pikv_engine_attach_nccl(self.h, buf))

    def local_attended(self) -> int:
        return int(lib().pikv_local_attended(self.h))

    def stream_handle(self) -> int:
        return int(lib().pikv_engine_stream(self.h) or 0)


__all__ = ["Engine", "EngineConfig", "EvictionRecord", "PikvError", "ShardId", "attention",
           "dequantize", "lowrank_decode", "lowrank_encode", "quantize", "select_evictions",
           "shard_assign", "_capi"]


class EngineGroup:
    """B streams split into ``n_micro`` engines pipelined on one GPU
    (include/pikv_b200.h, pikv_group_*): micro-batch m's control plane and
    fold-back overlap the other micro-batches' attention.  No reference
    counterpart; each stream still runs Engine::step (pipeline.cpp:213-351)."""

    def __init__(self, cfg: EngineConfig, n_micro: int = 2, attend_sms: int = 0, device: int = 0):
        import dataclasses
        self.cfg = cfg
        self._c = cfg.to_c()
        h = ctypes.c_void_p()
        check(lib().pikv_group_create(ctypes.byref(self._c), n_micro, attend_sms, device,
                                      ctypes.byref(h)))
        self.h, self.n, self.device = h, n_micro, device
        self.B, self.dp, self.d = cfg.batch, cfg.stored_width, cfg.model.d
        self.Bm = cfg.batch // n_micro
        mcfg = dataclasses.replace(cfg, batch=self.Bm)
        self.engines = [Engine._borrowed(mcfg, lib().pikv_group_engine(h, m), device)
                        for m in range(n_micro)]

    def close(self):
        h, self.h = getattr(self, "h", None), None
        if h:
            for e in self.engines:
                e.h = None
            try:
                lib().pikv_group_destroy(h)
            except (AttributeError, TypeError):
                pass

    __del__ = close

    def step(self, q, k, v, saliency=None, y=None):
        """One step of all B streams on full-batch device tensors (no host wait)."""
        if y is None:
            y = torch.empty(self.B, self.dp, dtype=torch.float32, device="cuda")
        cur = torch.cuda.current_stream()
        for e in self.engines:
            e.external_stream().wait_stream(cur)
        check(lib().pikv_group_step(self.h, _ptr(q), _ptr(k), _ptr(v), _ptr(saliency), _ptr(y)))
        for e in self.engines:
            cur.wait_stream(e.external_stream())
        return y

    def submit(self, m: int, q, k, v, saliency=None, y=None, host: bool = False):
        """Enqueue micro-batch m's step (raw pointers or tensors / arrays)."""
        conv = (lambda a: a if isinstance(a, int) or a is None else
                (a.ctypes.data if isinstance(a, np.ndarray) else a.data_ptr()))
        check(lib().pikv_group_submit(self.h, m, conv(q), conv(k), conv(v), conv(saliency),
                                      conv(y), int(host)))

    def wait(self, m: int):
        check(lib().pikv_group_wait(self.h, m))

    def join(self):
        check(lib().pikv_group_join(self.h))

    def sync(self):
        check(lib().pikv_group_sync(self.h))

    def set_timing(self, on: bool):
        check(lib().pikv_group_set_timing(self.h, int(on)))

    def read_timing(self):
        ms, n = ctypes.c_double(), ctypes.c_int32()
        check(lib().pikv_group_read_timing(self.h, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def attention_partition(self) -> bool:
        """True when the attention runs in its own green-context SM partition."""
        return bool(lib().pikv_group_attention_partition(self.h))

    def read_timing_union(self):
        """(summed attention launch ms, ms any attention launch was in flight, launches)."""
        tot, uni, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int32()
        check(lib().pikv_group_read_timing_union(self.h, ctypes.byref(tot), ctypes.byref(uni), ctypes.byref(n)))
        return tot.value, uni.value, n.value

    def prefill_synthetic(self, tokens: int, seed: int = 1):
        for m, e in enumerate(self.engines):
            e.prefill_synthetic(tokens, seed=seed + 7919 * m)

    def set_codec(self, basis=None, bias=None, kept=None):
        for e in self.engines:
            e.set_codec(basis, bias, kept)

    def kernel_launches(self) -> int:
        return sum(e.kernel_launches() for e in self.engines)

    def attach_nccl(self, uids):
        """One communicator per micro-batch (uids: n_micro unique ids)."""
        buf = ctypes.create_string_buffer(b"".join(bytes(u) for u in uids), 128 * self.n)
        check(lib().pikv_group_attach_nccl(self.h, buf))

    def read_step(self):
        """Concatenated (experts, gates, logits, summaries) over micro-batches."""
        parts = [e.read_step() for e in self.engines]
        return (np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]),
                np.concatenate([p[2] for p in parts]), sum((list(p[3]) for p in parts), []))
