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
from .graph import batch_from_v3, pack_batch_v3


class EpochRunner:
    """Graph-captured epoch of ``model_forward`` over ``batches``."""

    def __init__(self, model: ModelConfig, batches: list, *, jump: bool = True, reuse: str = "cross-tile",
                 stream: torch.cuda.Stream | None = None, rescan: bool = True, external_refresh: bool = False):
        self.model = model
        self.batches = list(batches)
        self.jump, self.reuse = jump, reuse
        # The zero-tile schedule is computed once per batch and cached on the adjacency,
        # as the reference caches scan_zero_tiles on the operand (bitgemm.py:222-233).
        # rescan=True re-gathers and re-expands the adjacency blocks from the current
        # words inside every epoch (new data each step, e2e path).
        self.rescan = rescan
        self.external_refresh = external_refresh   # the caller's pre() re-expands the blocks
        self.stream = stream or torch.cuda.Stream()
        self.graph = None
        self.logits = None
        self._keep = []

    def _forward_all(self, verify: bool):
        if self.rescan and not self.external_refresh:
            from .tiled import GroupedRefresh, blocked
            blks = [blocked(b.adjacency) for b in self.batches]
            if all(not getattr(k, "_gather", True) for k in blks):
                # shipped blocks (QGT3 views): one grouped expansion + degrees launch
                if getattr(self, "_grouped", None) is None:
                    self._grouped = GroupedRefresh(blks)
                self._grouped.run()
            else:
                for k in blks:                # new words each step: re-gather + re-expand the blocks
                    k.refresh()
        return model_forward_group(self.batches, self.model, jump=self.jump, reuse=self.reuse, verify=verify)

    def capture(self, pre=None, post=None, stamps: bool = False):
        """Capture the epoch; ``pre()`` / ``post(logits)`` are captured before / after it
        (HostEpochRunner: the H2D of the step's images and the D2H of the logits).
        ``stamps``: every tiled GEMM CTA records %globaltimer at entry/exit (bench.py's
        in-graph kernel durations; CUDA events cannot sit between a graph's kernels)."""
        from . import bitgemm
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
                self.stamps = []
                if stamps:
                    bitgemm.PHASE_HOOK = self.stamps
                from . import tiled
                n0 = tiled.LAUNCHES
                with torch.cuda.graph(self.graph, stream=self.stream):
                    if pre is not None:
                        pre()
                    self.slabs.reset()              # one slab-reset kernel per epoch
                    self.logits = self._forward_all(verify=False)
                    if post is not None:
                        post(self.logits)
                self.gemm_launches = tiled.LAUNCHES - n0
            except BaseException:
                N.STATIC_COPIES.clear()         # tables of a failed capture must never be copied later
                raise
            finally:
                N.ALLOC = N.TorchAlloc()
                bitgemm.PHASE_HOOK = None
            N.flush_static_copies()
        self._checks = list(getattr(self.model, "_pending_checks", []))
        return self

    def run(self):
        """Replay one epoch on the runner's stream (asynchronous)."""
        self.graph.replay()
        return self.logits

    def kernel_spans(self):
        """[(duration_ms, algorithmic_ops)] of the tiled GEMM launches of the LAST replay
        (capture(stamps=True)), on %globaltimer: from the later of the launch's first CTA
        entry and the previous GEMM launch's last CTA exit, to this launch's last CTA exit.
        With programmatic dependent launch a grid's CTAs enter while its predecessor is
        still running and wait in griddepcontrol.wait; counting from the predecessor's end
        keeps overlapped spans from being counted twice (the durations sum to the GEMM
        window of the epoch)."""
        out = []
        prev_end = None
        for st, work in self.stamps:
            s = st.cpu().numpy()
            s = s[s[:, 0] > 0]
            if len(s):
                begin, end = s[:, 0].min(), s[:, 5].max()
                if prev_end is not None:
                    begin = max(begin, prev_end)
                out.append(((end - begin) / 1e6, work))
                prev_end = end
        return out

    def kernel_launches_per_epoch(self) -> int:
        """Native (libqgtc_b200) kernels per epoch: the slab reset, 1 grouped entry
        conversion and the GEMM launches of the captured graph (2 per layer, fewer where
        stage pairs are chained); with rescan, per batch the block expansion (+ the gather
        from dense words unless the blocks were shipped, QGT3)."""
        from .tiled import blocked
        gemms = getattr(self, "gemm_launches", None)
        if gemms is None:
            gemms = 2 * len(self.model.layers)
        per_epoch = 2 + gemms
        if self.rescan:
            blks = [blocked(b.adjacency) for b in self.batches]
            if all(not getattr(k, "_gather", True) for k in blks):
                per_epoch += 1                                      # grouped expansion
            else:
                per_epoch += 2 * len(blks)
        return per_epoch


class HostEpochRunner:
    """End-to-end epoch as ONE CUDA graph: pinned host QGT3 images -> one H2D ->
    block expansion + the epoch -> one D2H of the fp64 logits into pinned memory.

    QGT3 (graph.pack_batch_v3) ships only the non-zero 128x128 adjacency blocks,
    so the H2D carries the zero-tile-jumping schedule instead of the dense bits."""

    def __init__(self, model: ModelConfig, batches: list, chunks: int | None = None, **kw):
        self.model = model
        images = [pack_batch_v3(b) for b in batches]
        self.offsets = np.cumsum([0] + [len(im) for im in images])
        self.host = torch.empty(int(self.offsets[-1]), dtype=torch.uint8).pin_memory()
        self.load(images)
        self.device = torch.empty_like(self.host, device=N.device())
        self.device.copy_(self.host)
        views = [batch_from_v3(im, self.device, int(o)) for im, o in zip(images, self.offsets)]
        rows = sum(v.total_nodes for v in views)
        self.classes = model.layers[-1].out_dim
        self.out_host = torch.empty((rows, self.classes), dtype=torch.float64).pin_memory()
        self.h2d_bytes = int(self.offsets[-1])
        self.d2h_bytes = rows * self.classes * 8
        # multi-batch epochs: pipeline the H2D (copy engine 1), the compute and the D2H (copy
        # engine 2) over chunks of batches -- PCIe is full duplex, so the input and output
        # transfers of different chunks overlap each other and the compute
        auto = 1 if len(views) < 8 else (4 if len(views) < 64 else 8)
        k = chunks if chunks is not None else auto
        self.chunks = max(1, min(k, len(views)))
        from .engine import UPDATE_THEN_AGGREGATE
        if self.chunks > 1:
            self._capture_pipelined(views)
        elif model.layers[0].order != UPDATE_THEN_AGGREGATE:
            # aggregate-first (GCN): the first GEMM needs the blocks -> nothing to overlap
            self.inner = EpochRunner(model, views, rescan=True, **kw).capture(pre=self._h2d, post=self._d2h)
        else:
            # split H2D: the feature sections first on the compute stream (entry conversion
            # and a GIN layer's update GEMM need only them); the schedule + adjacency blocks
            # on a side stream (second copy engine) with the block expansion behind them --
            # the first aggregation GEMM joins it (tiled.PENDING_JOIN)
            from .graph import v3_feature_offset
            from .tiled import GroupedRefresh, blocked
            self._feat_off = [int(o) + v3_feature_offset(im) for im, o in zip(images, self.offsets)]
            self._grouped = GroupedRefresh([blocked(v.adjacency) for v in views])
            self._grouped.run()                       # degrees valid for the eager recording pass
            self._s_in = torch.cuda.Stream()
            self.inner = EpochRunner(model, views, rescan=True, external_refresh=True, **kw).capture(
                pre=self._h2d_split, post=self._d2h_join)

    def _capture_pipelined(self, views):
        from .engine import _prepared, model_forward_group
        from .tiled import GroupedRefresh, blocked, weight_tiles
        groups = [list(g) for g in np.array_split(np.arange(len(views)), self.chunks)]
        _prepared(self.model)
        for ly, prep in zip(self.model.layers, _prepared(self.model)):
            weight_tiles(ly, prep)
        refresh = [GroupedRefresh([blocked(views[i].adjacency) for i in g]) for g in groups]
        row0 = np.cumsum([0] + [v.total_nodes for v in views])
        self._stream = torch.cuda.Stream()
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

        def forward(capturing: bool):
            outs_all = []
            ev_in = [torch.cuda.Event() for _ in groups]
            if capturing:
                with torch.cuda.stream(s_in):
                    s_in.wait_stream(self._stream)
                    for gi, g in enumerate(groups):
                        a, b = int(self.offsets[g[0]]), int(self.offsets[g[-1] + 1])
                        self.device[a:b].copy_(self.host[a:b], non_blocking=True)
                        ev_in[gi].record(s_in)
            for gi, g in enumerate(groups):
                if capturing:
                    self._stream.wait_event(ev_in[gi])
                refresh[gi].run()
                outs = model_forward_group([views[i] for i in g], self.model, verify=not capturing)
                outs_all += outs
                if capturing:
                    done = torch.cuda.Event()
                    done.record(self._stream)
                    with torch.cuda.stream(s_out):
                        s_out.wait_event(done)
                        self._copy_rows(outs, int(row0[g[0]]))
            if capturing:
                self._stream.wait_stream(s_in)
                self._stream.wait_stream(s_out)
            return outs_all

        with torch.cuda.stream(self._stream):
            plan = N.SlabPlan()
            N.ALLOC = plan
            try:
                forward(False)
            finally:
                N.ALLOC = N.TorchAlloc()
            torch.cuda.synchronize()
            self._slabs = N.SlabAlloc(plan)
            self._graph = torch.cuda.CUDAGraph()
            N.ALLOC = self._slabs
            try:
                with torch.cuda.graph(self._graph, stream=self._stream):
                    self._slabs.reset()
                    self._logits = forward(True)
            except BaseException:
                N.STATIC_COPIES.clear()
                raise
            finally:
                N.ALLOC = N.TorchAlloc()
            N.flush_static_copies()
        self.inner = None
        self._keep = (refresh, s_in, s_out)

    def _h2d(self):
        # the step's single H2D through the C-ABI (qg_batch_h2d; a memcpy node in the graph)
        N.check(N.lib().qg_batch_h2d(self.host.data_ptr(), self.host.numel(), self.device.data_ptr(), N.stream()),
                "qg_batch_h2d")

    def _h2d_split(self):
        from . import tiled
        main = torch.cuda.current_stream()
        self._s_in.wait_stream(main)
        for i, f0 in enumerate(self._feat_off):
            end = int(self.offsets[i + 1])
            if end > f0:
                self.device[f0:end].copy_(self.host[f0:end], non_blocking=True)
        with torch.cuda.stream(self._s_in):
            for i, f0 in enumerate(self._feat_off):
                a = int(self.offsets[i])
                self.device[a:f0].copy_(self.host[a:f0], non_blocking=True)
            self._grouped.run()
            ev = torch.cuda.Event()
            ev.record(self._s_in)
        tiled.PENDING_JOIN = ev

    def _d2h_join(self, outs):
        from . import tiled
        tiled.PENDING_JOIN = None
        torch.cuda.current_stream().wait_stream(self._s_in)      # side stream rejoins (no-op if joined)
        self._copy_rows(outs, 0)

    def _d2h(self, outs):
        self._copy_rows(outs, 0)

    def _copy_rows(self, outs, row0: int):
        """D2H of consecutive batches' logits into out_host[row0:]: the engine writes a
        launch's logits into one allocation (row-contiguous, batch order), so one strided
        view over it -> ONE copy."""
        rows = sum(o.shape[0] for o in outs)
        contiguous = bool(outs) and all(o.is_contiguous() for o in outs) and all(
            b.data_ptr() == a.data_ptr() + a.numel() * a.element_size() for a, b in zip(outs, outs[1:]))
        if contiguous:
            whole = outs[0].as_strided((rows, self.out_host.shape[1]), (self.out_host.shape[1], 1))
            self.out_host[row0:row0 + rows].copy_(whole, non_blocking=True)
            return
        r = row0
        for o in outs:
            self.out_host[r:r + o.shape[0]].copy_(o, non_blocking=True)
            r += o.shape[0]

    @property
    def stream(self):
        return self.inner.stream if self.inner is not None else self._stream

    def load(self, images) -> None:
        """Place a step's QGT3 images into the pinned staging area (host memcpy)."""
        for im, o in zip(images, self.offsets):
            self.host[int(o):int(o) + len(im)] = torch.frombuffer(bytearray(im), dtype=torch.uint8)

    def run_host(self) -> torch.Tensor:
        """H2D + epoch + D2H: one graph launch on the runner's stream; returns the pinned logits
        (valid after the stream synchronises)."""
        with torch.cuda.stream(self.stream):
            if self.inner is not None:
                self.inner.run()
            else:
                self._graph.replay()
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
            except BaseException:
                N.STATIC_COPIES.clear()
                raise
            finally:
                N.ALLOC = N.TorchAlloc()
            N.flush_static_copies()

    def run(self):
        self.graph.replay()
        return self.result
