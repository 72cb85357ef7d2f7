# SPDX-License-Identifier: Apache-2.0
"""Multi-rank decode step: experts sharded over ranks, partial softmax states
merged across ranks.

Placement follows the reference's own shard_assign (kvstore.cpp:14-30): with
G logical devices and G ranks, device g lives on rank g.  Routing is
replicated (W_r is identical on every rank), each rank inserts, evicts
(budgets are per device, scheduler.cpp:269) and attends only over its own
shards, and the one real exchange of the path is the log-sum-exp merge
(SURVEY §8 a14/e): every rank all-gathers the per-stream exchange records
(m, l, o[H][d'h], per-expert hit counts, step counters) and finishes the
step locally (global y, global (m, l) for the alpha fold-back, misses).

On GPUs the collective lives inside the library: ``attach_nccl`` creates
the engine's NCCL communicator (rank 0's unique id broadcast over the
caller's process group) and every ``Engine.step`` then runs the whole
sharded step -- the all-gather enqueued on the engine stream inside the
captured step graph.  ``ShardedStepper`` drives the same exchange through
pikv_step_local / pikv_step_finish with torch.distributed as the transport
(gloo: the multi-process tests, staged through host memory).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class _DevBuf:
    """Zero-copy torch view of an engine-owned device buffer."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


def device_view(ptr: int, nbytes: int) -> torch.Tensor:
    return torch.as_tensor(_DevBuf(ptr, nbytes), device="cuda")


def all_gather_bytes(out: torch.Tensor, local: torch.Tensor, group=None):
    """out[r * n:(r+1) * n] = local of rank r.  NCCL gathers device buffers in
    place; gloo (CPU tests, or a single-GPU rehearsal of the multi-rank path)
    stages device buffers through host memory."""
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, local, group=group)
        return out
    n = local.numel()
    loc = local.cpu() if local.is_cuda else local
    host = torch.empty(out.numel(), dtype=out.dtype)
    parts = [host[r * n:(r + 1) * n] for r in range(dist.get_world_size(group))]
    dist.all_gather(parts, loc, group=group)
    out.copy_(host)
    return out


def attach_nccl(engine, group=None, n_comms: int = 1):
    """Create the library-owned NCCL communicator(s) of `engine` (an Engine,
    or an EngineGroup with one communicator per micro-batch): rank 0 draws
    the unique ids, the process group broadcasts them."""
    from .engine import Engine
    ids = [Engine.nccl_unique_id() for _ in range(n_comms)] if dist.get_rank(group) == 0 else None
    box = [ids]
    dist.broadcast_object_list(box, src=0, group=group)
    ids = box[0]
    if n_comms == 1 and hasattr(engine, "attach_nccl") and not hasattr(engine, "engines"):
        engine.attach_nccl(ids[0])
    else:
        engine.attach_nccl(ids)
    return engine


class ShardedStepper:
    """Drive one rank's engine through the sharded step:
    step_local -> all-gather(exchange) -> step_finish.

    ``engine`` provides exchange_bytes(), step_local(q, k, v, saliency) -> ptr
    or tensor, step_finish(gathered, y) and external_stream() (or None)."""

    def __init__(self, engine, group=None):
        self.eng = engine
        self.group = group
        self.world = dist.get_world_size(group)
        self.nbytes = engine.exchange_bytes()
        on_gpu = engine.external_stream() is not None
        dev = "cuda" if on_gpu else "cpu"
        self.gathered = torch.empty(self.world * self.nbytes, dtype=torch.uint8, device=dev)

    def step(self, q, k, v, y=None, saliency=None):
        es = self.eng.external_stream()
        if es is not None:
            es.wait_stream(torch.cuda.current_stream())
        local = self.eng.step_local(q, k, v, saliency)
        if isinstance(local, int):
            local = device_view(local, self.nbytes)
        if es is not None:
            with torch.cuda.stream(es):
                all_gather_bytes(self.gathered, local, self.group)
        else:
            all_gather_bytes(self.gathered, local, self.group)
        y = self.eng.step_finish(self.gathered, y)
        if es is not None:
            torch.cuda.current_stream().wait_stream(es)
        return y
