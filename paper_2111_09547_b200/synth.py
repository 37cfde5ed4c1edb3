"""Synthetic workloads shaped like BASELINE.json's configs.

Graphs are planted partitions: P equal parts, ~80% of the undirected edges
inside a part (sampled uniformly), the rest across parts -- which batching
drops anyway (graph.py:337).  Partitions are supplied directly (the METIS
import path, graph.py:232-256), so no partitioner runs.  Features are
uniform [0, 1) (cli.py:160); weights U(-0.5, 0.5), bias U(-0.1, 0.1)
(engine.py:418-420); grids are calibrated on batch 0 (cli.py:209).

``planted_batches`` builds each batch directly from its parts' local edges on
the GPU (equivalent to ``build_batch`` on the planted graph, checked by
tests/test_gpu_synth.py) so the 2.4M-node config does not need a global edge sort.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .bitpack import COLUMN_WISE, ROW_WISE, BitPlaneStack, PackedBitMatrix, pad8, pad128
from .engine import calibrate_model, gcn_model, gin_model
from .graph import SubgraphBatch
from .quantize import QuantParams, quantize_pack_device
from .synth_host import (CONFIGS, GraphConfig, batch_edge_list, batch_part_sizes, host_batch,  # noqa: F401
                         intra_edges_per_part, num_batches, part_bounds, with_bits)


def planted_batches(cfg: GraphConfig, seed: int = 0, batch_ids=None, features_dtype=np.float32):
    """Build SubgraphBatches of the planted graph on the GPU.

    Returns (batches, features_per_batch_host, x_params).  Node ids are
    contiguous per part (part p owns [bounds[p], bounds[p+1])), parts are
    batched in order, ``parts_per_batch`` at a time (cli.py:179-186).  The host
    inputs come from ``synth_host.host_batch`` (shared with the reference arm).
    """
    bounds = part_bounds(cfg)
    ids = range(num_batches(cfg)) if batch_ids is None else batch_ids
    x_params = QuantParams(0.0, 1.0, cfg.bits)   # features U[0,1): grid [min, max) ~ [0, 1)
    batches, feats = [], []
    for b in ids:
        edges, boundaries, x = host_batch(cfg, seed, b, features_dtype)
        total = int(boundaries[-1])
        el = batch_edge_list(edges, boundaries)
        src = N.to_device(np.ascontiguousarray(el[:, 0]))
        dst = N.to_device(np.ascontiguousarray(el[:, 1]))
        pr, pc = pad8(total), pad128(total)
        words = torch.zeros(pr * pc // 32, dtype=torch.int32, device=N.device())
        N.call("qg_edges_to_bits", N.ptr(src), N.ptr(dst), src.numel(), total, N.ptr(words), pr, pc, N.stream())
        adj = PackedBitMatrix(COLUMN_WISE, total, total, pr, pc, words)
        r = quantize_pack_device(x, x_params, N.ROW_WISE_ID, 8, row_sums=True)
        fst = BitPlaneStack._wrap(ROW_WISE, total, cfg.in_dim, r["pr"], r["pc"], r["planes"])
        p0 = b * cfg.parts_per_batch
        lo = int(bounds[p0])
        batches.append(SubgraphBatch(node_ids=np.arange(lo, lo + total), adjacency=adj, features=fst,
                                     boundaries=boundaries, x_params=x_params, feat_row_sums=r["row_sums"]))
        feats.append(x)
    return batches, feats, x_params


def make_model(cfg: GraphConfig, seed: int = 0):
    builder = gcn_model if cfg.model == "gcn" else gin_model
    return builder(cfg.in_dim, cfg.classes, hidden_dim=cfg.hidden, num_layers=cfg.layers,
                   feature_bits=cfg.bits, weight_bits=cfg.wbits, seed=seed)


def calibrated_model(cfg: GraphConfig, batch0, feats0, seed: int = 0):
    model = make_model(cfg, seed)
    calibrate_model(model, batch0, feats0)
    return model


def bernoulli_adjacency(m: int, k: int, density: float, seed: int = 0, blocks: int = 1) -> PackedBitMatrix:
    """C5 adjacency: Bernoulli(density) bits, optionally restricted to ``blocks``
    equal diagonal blocks (to exercise zero-tile jumping).  Built on the GPU."""
    dev = N.device()
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    pr, pc = pad8(m), pad128(k)
    bits = (torch.rand((m, k), generator=g, device=dev) < density)
    if blocks > 1:
        rb = torch.arange(m, device=dev) * blocks // m
        cb = torch.arange(k, device=dev) * blocks // k
        bits &= rb[:, None] == cb[None, :]
    from .bitpack import _pack_device
    return _pack_device(bits.to(torch.uint8).unsqueeze(0), COLUMN_WISE, 8).planes[0]


def random_codes_stack(rows: int, cols: int, bits: int, orientation: str, seed: int = 0, pad_to: int = 8):
    """Uniform integer codes in [0, 2^bits) packed as planes (C5 X operand)."""
    dev = N.device()
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    codes = torch.randint(0, 1 << bits, (rows, cols), generator=g, device=dev, dtype=torch.int32).to(torch.uint8)
    oid = N.COLUMN_WISE_ID if orientation == COLUMN_WISE else N.ROW_WISE_ID
    from .bitpack import padded_dims
    pr, pc = padded_dims(rows, cols, orientation, pad_to)
    planes = torch.empty((bits, pr * pc // 32), dtype=torch.int32, device=dev)
    status = N.new_status()
    N.call("qg_quantize_pack", N.ptr(codes), N.SRC_U8, rows, cols, cols, 0.0, 1.0, bits, oid, pad_to,
           N.ptr(planes), None, None, None, N.ptr(status), N.stream())
    return BitPlaneStack._wrap(orientation, rows, cols, pr, pc, planes), codes
