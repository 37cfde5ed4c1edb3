"""Epoch runtime: one CUDA graph per epoch over a fixed set of batches.

The reference's timed region (cli.py:212-222) is ``for b in batches:
model_forward(b)``.  ``EpochRunner`` captures exactly that loop -- tile scan
(zero-tile-jumping schedule + degrees), the entry repack and the two fused
bit-GEMM launches per layer, for every batch -- into one CUDA graph, so a
whole epoch is a single ``cudaGraphLaunch`` with no Python or launch
overhead.

Two inputs modes:

* device-resident (``run()``): batches already in HBM;
* end to end (``run_host()``): the step's QGTB compound buffers are copied
  from pinned host memory into ONE device staging buffer (one H2D per
  epoch; batches are device views into it), the graph replays, and the fp64
  logits come back into pinned host memory (one D2H) -- all stream-ordered.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .engine import ModelConfig, _prepared, model_forward_group
from .graph import batch_from_v2, pack_batch_v2


class EpochRunner:
    """Graph-captured epoch of ``model_forward`` over ``batches``."""

    def __init__(self, model: ModelConfig, batches: list, *, jump: bool = True, reuse: str = "cross-tile",
                 stream: torch.cuda.Stream | None = None, rescan: bool = True):
        self.model = model
        self.batches = list(batches)
        self.jump, self.reuse = jump, reuse
        # The zero-tile schedule is computed once per batch and cached on the adjacency,
        # as the reference caches scan_zero_tiles on the operand (bitgemm.py:222-233).
        # rescan=True re-gathers and re-expands the adjacency blocks from the current
        # words inside every epoch (new data each step, e2e path).
        self.rescan = rescan
        self.stream = stream or torch.cuda.Stream()
        self.graph = None
        self.logits = None
        self._keep = []

    def _forward_all(self, verify: bool):
        if self.rescan:
            from .tiled import blocked
            for b in self.batches:            # new words each step: re-gather + re-expand the blocks
                blocked(b.adjacency).refresh()
        return model_forward_group(self.batches, self.model, jump=self.jump, reuse=self.reuse, verify=verify)

    def capture(self):
        _prepared(self.model)
        from .tiled import blocked, weight_tiles
        for b in self.batches:
            blocked(b.adjacency)              # zero-tile schedule (host-known) + blocks, outside the epoch
        for ly, prep in zip(self.model.layers, _prepared(self.model)):
            weight_tiles(ly, prep)
        with torch.cuda.stream(self.stream):
            plan = N.SlabPlan()
            N.ALLOC = plan
            try:
                self._forward_all(verify=True)      # eager warm-up: records the allocation sequence
            finally:
                N.ALLOC = N.TorchAlloc()
            torch.cuda.synchronize()
            self.slabs = N.SlabAlloc(plan)
            self.graph = torch.cuda.CUDAGraph()
            N.ALLOC = self.slabs
            try:
                with torch.cuda.graph(self.graph, stream=self.stream):
                    self.slabs.reset()              # 1 memset + 1 fill per epoch
                    self.logits = self._forward_all(verify=False)
            finally:
                N.ALLOC = N.TorchAlloc()
            N.flush_static_copies()
        self._checks = list(getattr(self.model, "_pending_checks", []))
        return self

    def run(self):
        """Replay one epoch on the runner's stream (asynchronous)."""
        self.graph.replay()
        return self.logits

    def kernel_launches_per_epoch(self) -> int:
        """Native kernels per epoch: per batch 2 (tile scan + schedule) + 1 entry code
        conversion + 2 fused GEMMs per layer."""
        per_epoch = 2 * len(self.model.layers) + 2 * len(self.batches)   # grouped GEMMs + entry conversions
        if self.rescan:
            per_epoch += 2 * len(self.batches)                              # block gather + expand
        return per_epoch


class HostEpochRunner:
    """End-to-end epoch: pinned host QGT2 images -> one H2D -> epoch graph -> one D2H."""

    def __init__(self, model: ModelConfig, batches: list, **kw):
        self.model = model
        images = [pack_batch_v2(b) for b in batches]
        self.offsets = np.cumsum([0] + [len(im) for im in images])
        self.host = torch.empty(int(self.offsets[-1]), dtype=torch.uint8).pin_memory()
        self.load(images)
        self.device = torch.empty_like(self.host, device=N.device())
        self.device.copy_(self.host)
        views = [batch_from_v2(im, self.device, int(o)) for im, o in zip(images, self.offsets)]
        self.inner = EpochRunner(model, views, rescan=True, **kw).capture()
        rows = sum(v.total_nodes for v in views)
        self.classes = model.layers[-1].out_dim
        self.out_host = torch.empty((rows, self.classes), dtype=torch.float64).pin_memory()
        self.h2d_bytes = int(self.offsets[-1])
        self.d2h_bytes = rows * self.classes * 8

    @property
    def stream(self):
        return self.inner.stream

    def load(self, images) -> None:
        """Place a step's QGT2 images into the pinned staging area (host memcpy)."""
        for im, o in zip(images, self.offsets):
            self.host[int(o):int(o) + len(im)] = torch.frombuffer(bytearray(im), dtype=torch.uint8)

    def run_host(self) -> torch.Tensor:
        """H2D + epoch graph + D2H on the runner's stream; returns the pinned logits."""
        with torch.cuda.stream(self.stream):
            self.device.copy_(self.host, non_blocking=True)
            outs = self.inner.run()
            r = 0
            for o in outs:
                self.out_host[r:r + o.shape[0]].copy_(o, non_blocking=True)
                r += o.shape[0]
        return self.out_host


class CapturedCall:
    """Any device-only call (e.g. ``tiled.bmm_reduced``) replayed as one CUDA graph.

    Same recipe as ``EpochRunner``: one eager run records the allocation
    sequence, the slabs then serve it so the captured graph owns its buffers
    (segment tables included, from pinned host slabs)."""

    def __init__(self, fn, stream: torch.cuda.Stream | None = None):
        self.fn = fn
        self.stream = stream or torch.cuda.Stream()
        with torch.cuda.stream(self.stream):
            plan = N.SlabPlan()
            N.ALLOC = plan
            try:
                fn()
            finally:
                N.ALLOC = N.TorchAlloc()
            torch.cuda.synchronize()
            self.slabs = N.SlabAlloc(plan)
            self.graph = torch.cuda.CUDAGraph()
            N.ALLOC = self.slabs
            try:
                with torch.cuda.graph(self.graph, stream=self.stream):
                    self.slabs.reset()
                    self.result = fn()
            finally:
                N.ALLOC = N.TorchAlloc()
            N.flush_static_copies()

    def run(self):
        self.graph.replay()
        return self.result
