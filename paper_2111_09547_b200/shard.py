"""Sharding subgraph batches over the GPUs of one box.

Subgraph batches are independent: block-diagonal, no cross-batch edges
(graph.py:313-314, 337), so an epoch shards with no data-path collective.
Each rank owns a set of batches (LPT on the estimated work, sum over parts of
n_p^2 * D * s), runs its own epoch graph over them, and the per-batch fp64
logits are gathered to rank 0 once per epoch with ONE collective
(``all_gather_into_tensor`` over NCCL/NVLink on the GPU, gloo in the CPU
tests).  Weights and calibrated grids are replicated: every rank prepares them
deterministically (engine.py:148-155).
"""

from __future__ import annotations

import heapq

import numpy as np
import torch


def batch_cost(part_sizes, in_dim: int, bits: int) -> float:
    """Estimated work of one batch: sum_p n_p^2 * D * s."""
    return float(sum(int(n) * int(n) for n in part_sizes)) * in_dim * bits


def assign_lpt(costs, world: int) -> list[list[int]]:
    """Longest-processing-time-first assignment of batch ids to ranks.

    Deterministic (ties broken by rank then batch id), so every rank computes the
    same plan without communicating.  Each rank's list is sorted ascending."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-float(costs[i]), i))
    heap = [(0.0, r) for r in range(world)]
    out = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + float(costs[i]), r))
    return [sorted(v) for v in out]


def imbalance(costs, plan) -> float:
    """max rank load / mean rank load (1.0 = perfect)."""
    loads = [sum(float(costs[i]) for i in ids) for ids in plan]
    mean = sum(loads) / max(len(loads), 1)
    return max(loads) / mean if mean > 0 else 1.0


class LogitGather:
    """Gather every rank's per-batch logits to rank 0 in global batch order.

    ``rows[b]`` = nodes of batch b (known on every rank from the plan), so each
    rank's shard is padded to the largest shard and ONE ``all_gather_into_tensor``
    moves the epoch's outputs; rank 0 scatters the padded shards back into batch
    order.  Buffers are allocated once (the gather can sit inside a timed loop)."""

    def __init__(self, plan, rows, classes: int, device, dtype=torch.float64, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = len(plan)
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.plan = plan
        self.rows = [int(r) for r in rows]
        self.shard_rows = [sum(self.rows[i] for i in ids) for ids in plan]
        self.pad = max(self.shard_rows) if self.shard_rows else 0
        self.classes = classes
        self.send = torch.zeros((max(self.pad, 1), classes), dtype=dtype, device=device)
        self.recv = torch.zeros((self.world * max(self.pad, 1), classes), dtype=dtype, device=device)
        starts = np.cumsum([0] + self.rows)
        self.global_start = starts[:-1]
        self.total_rows = int(starts[-1])

    def gather(self, local_outs) -> torch.Tensor | None:
        """local_outs: this rank's logits, one tensor per owned batch (plan order).
        Returns the full (total_rows, classes) logits on rank 0, None elsewhere."""
        r = 0
        for o in local_outs:
            self.send[r:r + o.shape[0]].copy_(o)
            r += o.shape[0]
        if self.world > 1:
            self.dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
        else:
            self.recv[:self.send.shape[0]].copy_(self.send)
        if self.rank != 0:
            return None
        return self.assemble(self.recv)

    def assemble(self, recv: torch.Tensor) -> torch.Tensor:
        full = torch.empty((self.total_rows, self.classes), dtype=recv.dtype, device=recv.device)
        stride = max(self.pad, 1)
        for rk, ids in enumerate(self.plan):
            off = rk * stride
            for b in ids:
                n = self.rows[b]
                g = int(self.global_start[b])
                full[g:g + n].copy_(recv[off:off + n])
                off += n
        return full
