# SPDX-License-Identifier: Apache-2.0
"""Multi-process (gloo, world_size 2) test of the sharded step's host logic:
paper_2508_06526_b200.parallel.ShardedStepper all-gathers each rank's
exchange record and hands the gathered buffer to step_finish.

The engine here is a CPU stand-in with the product's exchange record layout
(ExchangeLayout in csrc/pikv_dev.cuh: o[H][d'h], m[H], l[H] in base 2, hit
counts, stats): each rank attends over its own part of the entries and its
finish merges the partial softmax states.  The merged output
must equal one softmax over the union of the entries (fp64 oracle)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_06526_b200.parallel import ShardedStepper

B, H, DH, K = 3, 4, 8, 2
LOG2E = 1.4426950408889634


def layout():
    o_off = 0
    m_off = o_off + 4 * H * DH
    l_off = m_off + 4 * H
    f_off = l_off + 4 * H
    st_off = f_off + 4 * K
    per = ((st_off + 16 + 15) // 16) * 16
    return o_off, m_off, l_off, f_off, st_off, per


class CpuShardEngine:
    """Rank-local partial attention + the finish merge, in numpy."""

    def __init__(self, q, keys, values, owner, rank):
        self.q, self.keys, self.values, self.owner, self.rank = q, keys, values, owner, rank
        self.layout = layout()

    def exchange_bytes(self):
        return B * self.layout[5]

    def external_stream(self):
        return None

    def step_local(self, q, k, v, saliency):
        o_off, m_off, l_off, f_off, st_off, per = self.layout
        buf = np.zeros(B * per, dtype=np.uint8)
        for s in range(B):
            rec = buf[s * per:(s + 1) * per]
            mine = [i for i in range(len(self.keys[s])) if self.owner[s][i] == self.rank]
            o = np.zeros((H, DH), dtype=np.float32)
            m = np.full(H, -np.inf, dtype=np.float32)
            l_ = np.zeros(H, dtype=np.float32)
            for h in range(H):
                if mine:
                    sc = np.array([self.q[s][h] @ self.keys[s][i][h] for i in mine]) / np.sqrt(DH) * LOG2E
                    m[h] = sc.max()
                    p = np.exp2(sc - m[h])
                    l_[h] = p.sum()
                    o[h] = sum(pi * self.values[s][i][h] for pi, i in zip(p, mine))
            rec[o_off:m_off] = np.frombuffer(o.astype(np.float32).tobytes(), np.uint8)
            rec[m_off:l_off] = np.frombuffer(m.tobytes(), np.uint8)
            rec[l_off:f_off] = np.frombuffer(l_.tobytes(), np.uint8)
            rec[f_off:st_off] = np.frombuffer(np.array([len(mine), 0], np.int32).tobytes(), np.uint8)
        return torch.from_numpy(buf)

    def step_finish(self, gathered, y=None):  # k_finish_merge restated
        o_off, m_off, l_off, f_off, st_off, per = self.layout
        g = gathered.numpy()
        world = g.size // (B * per)
        out = np.zeros((B, H, DH))
        for s in range(B):
            recs = [g[r * B * per + s * per: r * B * per + (s + 1) * per] for r in range(world)]
            for h in range(H):
                ms = [np.frombuffer(rc[m_off:l_off].tobytes(), np.float32)[h] for rc in recs]
                M = max(ms)
                if M == -np.inf:
                    continue
                L = 0.0
                acc = np.zeros(DH)
                for rc, mr in zip(recs, ms):
                    if mr == -np.inf:
                        continue
                    f = 2.0 ** (mr - M)
                    L += np.frombuffer(rc[l_off:f_off].tobytes(), np.float32)[h] * f
                    acc += np.frombuffer(rc[o_off:m_off].tobytes(), np.float32).reshape(H, DH)[h] * f
                out[s, h] = acc / L
        return out


def _worker(rank, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    rng = np.random.default_rng(5)  # same data on both ranks
    n = [7, 0, 12]
    q = rng.standard_normal((B, H, DH))
    keys = [rng.standard_normal((n[s], H, DH)) for s in range(B)]
    values = [rng.standard_normal((n[s], H, DH)) for s in range(B)]
    owner = [rng.integers(0, 2, n[s]) for s in range(B)]  # expert placement per entry
    eng = CpuShardEngine(q, keys, values, owner, rank)
    y = ShardedStepper(eng).step(None, None, None)
    # one softmax over the union (pipeline.cpp:59-85 per head, fp64)
    want = np.zeros((B, H, DH))
    for s in range(B):
        for h in range(H):
            if n[s] == 0:
                continue
            sc = np.array([q[s][h] @ keys[s][i][h] for i in range(n[s])]) / np.sqrt(DH)
            a = np.exp(sc - sc.max())
            a /= a.sum()
            want[s, h] = sum(a[i] * values[s][i][h] for i in range(n[s]))
    result_q.put((rank, float(np.max(np.abs(y - want)))))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def test_sharded_stepper_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert [r for r, _ in res] == [0, 1]
    for _, err in res:
        assert err < 1e-5, err
