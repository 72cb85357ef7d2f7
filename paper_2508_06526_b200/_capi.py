# SPDX-License-Identifier: Apache-2.0
"""ctypes binding of libpikv_b200.so (include/pikv_b200.h).

The library is the product; this module only declares signatures.  Loading
fails loudly when the shared object is missing -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

from .config import PikvConfigC

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpikv_b200.so")

c_i32, c_i64, c_u64, c_f64, c_vp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                    ctypes.c_double, ctypes.c_void_p)
P = ctypes.POINTER

ERRORS = {
    1: "InvalidArgument", 2: "InvalidConfig", 3: "InvalidEntry", 4: "NumericalError",
    5: "CodecMismatch", 6: "NotFitted", 7: "InsufficientCalibration", 8: "InvalidComparison",
    9: "IoError", 10: "CudaError", 11: "NcclError", 12: "OutOfMemory",
}


class PikvEvictRecord(ctypes.Structure):
    _fields_ = [("step", c_u64), ("entry_id", c_u64), ("token_id", c_i64), ("expert_id", c_i32),
                ("device", c_i32), ("score", c_f64), ("reason", c_i32), ("stream", c_i32)]


class PikvEntry(ctypes.Structure):
    """pikv_entry: KVEntry identity + EntryMeta (types.hpp:11-34)."""
    _fields_ = [("id", c_u64), ("shard_seq", c_u64), ("token_id", c_i64), ("expert_id", c_i32),
                ("has_layers", c_i32), ("insert_step", c_u64), ("last_access_step", c_u64),
                ("freq", c_u64), ("attn_mass", c_f64)]


class PikvStepSummary(ctypes.Structure):
    _fields_ = [("step", c_u64), ("inserts", c_i32), ("hits", c_i32), ("lookups", c_i32),
                ("n_attended", c_i32), ("fetch_elements", c_i64), ("n_evictions", c_i32),
                ("pages_before", c_i32), ("pages_after", c_i32), ("error", c_i32)]


# name -> (restype, argtypes); every symbol include/pikv_b200.h declares.
SIGNATURES = {
    "pikv_version": (ctypes.c_char_p, []),
    "pikv_last_error": (ctypes.c_char_p, []),
    "pikv_config_size": (ctypes.c_int, []),
    "pikv_config_default": (None, [P(PikvConfigC)]),
    "pikv_shard_assign": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp,
                                         c_vp, c_vp]),
    "pikv_select_evictions": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_i32, c_f64, c_vp,
                                             c_vp, c_vp]),
    "pikv_attention": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp]),
    "pikv_quantize": (ctypes.c_int, [c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_vp]),
    "pikv_dequantize": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_i32, c_vp]),
    "pikv_lowrank_encode": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_vp]),
    "pikv_lowrank_decode": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_vp]),
    "pikv_shard_assign_host": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp,
                                              c_vp, c_vp]),
    "pikv_select_evictions_host": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_i32, c_f64, c_vp,
                                                  c_vp, c_vp]),
    "pikv_attention_host": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp]),
    "pikv_engine_create": (ctypes.c_int, [P(PikvConfigC), c_i32, P(c_vp)]),
    "pikv_engine_destroy": (ctypes.c_int, [c_vp]),
    "pikv_engine_stream": (c_vp, [c_vp]),
    "pikv_set_router_matrix_host": (ctypes.c_int, [c_vp, c_vp]),
    "pikv_set_codec_host": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "pikv_step": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pikv_step_host": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pikv_exchange_bytes": (c_i64, [c_vp]),
    "pikv_step_local": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, P(c_vp)]),
    "pikv_step_finish": (ctypes.c_int, [c_vp, c_vp, c_vp]),
    "pikv_prefill_synthetic": (ctypes.c_int, [c_vp, c_i64, c_u64]),
    "pikv_fill_synthetic": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_u64]),
    "pikv_sync": (ctypes.c_int, [c_vp]),
    "pikv_read_step_host": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pikv_read_evictions_host": (ctypes.c_int, [c_vp, c_vp, c_i32, P(c_i32)]),
    "pikv_read_attended_host": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp, c_vp, c_i32, P(c_i32)]),
    "pikv_step_embed": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "pikv_step_embed_host": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "pikv_set_encoder_host": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "pikv_insert_bulk": (ctypes.c_int, [c_vp, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, P(c_i64)]),
    "pikv_insert_bulk_host": (ctypes.c_int, [c_vp, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, P(c_i64)]),
    "pikv_generate_trace": (ctypes.c_int, [c_u64, c_i32, c_i32, c_f64, c_u64, c_i32, c_vp, c_vp,
                                           c_vp]),
    "pikv_snapshot_host": (ctypes.c_int, [c_vp, c_i32, ctypes.c_int64, c_vp, ctypes.c_int64,
                                          P(ctypes.c_int64)]),
    "pikv_slot_count": (c_i64, [c_vp]),
    "pikv_read_slots_host": (ctypes.c_int, [c_vp, c_i32] + [c_vp] * 9),
    "pikv_write_attn_mass_host": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp]),
    "pikv_read_entries_host": (ctypes.c_int, [c_vp, c_i32, c_vp, c_i32, c_vp, c_vp]),
    "pikv_read_router_state_host": (ctypes.c_int, [c_vp, c_i32] + [c_vp] * 6),
    "pikv_read_sched_state_host": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp, c_vp]),
    "pikv_store_stats_host": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "pikv_pool_pages_in_use": (c_i64, [c_vp]),
    "pikv_entry_bytes": (c_i64, [c_vp]),
    "pikv_kernel_launches": (c_i64, [c_vp]),
    "pikv_set_profiling": (ctypes.c_int, [c_vp, c_i32]),
    "pikv_read_profile_host": (ctypes.c_int, [c_vp, c_vp, c_i32, P(c_i32)]),
    "pikv_group_create": (ctypes.c_int, [P(PikvConfigC), c_i32, c_i32, c_i32, P(c_vp)]),
    "pikv_group_destroy": (ctypes.c_int, [c_vp]),
    "pikv_group_size": (ctypes.c_int, [c_vp]),
    "pikv_group_engine": (c_vp, [c_vp, c_i32]),
    "pikv_group_submit": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32]),
    "pikv_group_wait": (ctypes.c_int, [c_vp, c_i32]),
    "pikv_group_step": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pikv_group_join": (ctypes.c_int, [c_vp]),
    "pikv_group_sync": (ctypes.c_int, [c_vp]),
    "pikv_group_set_timing": (ctypes.c_int, [c_vp, c_i32]),
    "pikv_group_read_timing": (ctypes.c_int, [c_vp, P(c_f64), P(c_i32)]),
    "pikv_group_read_timeline": (ctypes.c_int, [c_vp, P(c_f64), c_i32, P(c_i32)]),
    "pikv_group_read_timing_union": (ctypes.c_int, [c_vp, P(c_f64), P(c_f64), P(c_i32)]),
    "pikv_group_attention_partition": (ctypes.c_int, [c_vp]),
    "pikv_nccl_unique_id": (ctypes.c_int, [c_vp]),
    "pikv_engine_attach_nccl": (ctypes.c_int, [c_vp, c_vp]),
    "pikv_engine_set_nccl_comm": (ctypes.c_int, [c_vp, c_vp]),
    "pikv_local_attended": (c_i64, [c_vp]),
    "pikv_group_attach_nccl": (ctypes.c_int, [c_vp, c_vp]),
    # component API
    "pikv_update_config": (ctypes.c_int, [c_vp, P(PikvConfigC)]),
    "pikv_route_host": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "pikv_route_logits_host": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "pikv_record_miss": (ctypes.c_int, [c_vp, c_i32, c_i32]),
    "pikv_router_adapt": (ctypes.c_int, [c_vp, c_i32, c_vp, c_i32, c_f64]),
    "pikv_write_router_state_host": (ctypes.c_int, [c_vp, c_i32] + [c_vp] * 6),
    "pikv_write_sched_state_host": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp, c_vp]),
    "pikv_store_insert_host": (ctypes.c_int, [c_vp, c_i32, c_i32] + [c_vp] * 9),
    "pikv_store_retrieve_host": (ctypes.c_int, [c_vp, c_i32, c_vp, c_i32, c_i64, c_u64, c_vp, c_i32,
                                                P(c_i32), c_vp, P(c_i32)]),
    "pikv_store_erase_host": (ctypes.c_int, [c_vp, c_i32, c_u64, P(c_i32)]),
    "pikv_store_counters_host": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp]),
    "pikv_ring_live_host": (ctypes.c_int, [c_vp, c_i32, c_vp]),
    "pikv_score_entries_host": (ctypes.c_int, [P(PikvConfigC), c_vp, c_vp, c_i32, c_u64, c_vp]),
    "pikv_evict_host": (ctypes.c_int, [c_vp, c_i32, c_u64, c_vp, c_i32, P(c_i32), P(c_i32), P(c_i32)]),
    "pikv_observe_hits": (ctypes.c_int, [c_vp, c_i32, c_u64, c_u64]),
    "pikv_adakv_update": (ctypes.c_int, [c_vp, c_i32]),
    "pikv_attend_host": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp, c_i32, c_vp, c_vp]),
    "pikv_codec_encode": (ctypes.c_int, [c_i32] * 5 + [c_vp] * 5),
    "pikv_codec_decode": (ctypes.c_int, [c_i32] * 5 + [c_vp] * 5),
    "pikv_codec_encode_host": (ctypes.c_int, [c_i32] * 5 + [c_vp] * 5),
    "pikv_codec_decode_host": (ctypes.c_int, [c_i32] * 5 + [c_vp] * 5),
    "pikv_column_variance_host": (ctypes.c_int, [c_vp, c_i32, c_i32, c_vp]),
}

_LIB = None


class PikvError(RuntimeError):
    """Mirror of pikv::Error (errors.hpp:9); .kind names the reference class."""

    def __init__(self, code: int, msg: str):
        self.code = code
        self.kind = ERRORS.get(code, "Error")
        super().__init__("%s: %s" % (self.kind, msg))


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                "libpikv_b200.so not built (run python -m paper_2508_06526_b200.build); "
                "there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def check(rc: int):
    if rc != 0:
        raise PikvError(rc, lib().pikv_last_error().decode())
