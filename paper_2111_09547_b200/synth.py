"""Synthetic workloads shaped like BASELINE.json's configs.

Graphs are planted partitions: P equal parts, ~80% of the undirected edges
inside a part (sampled uniformly), the rest across parts -- which batching
drops anyway (graph.py:337).  Partitions are supplied directly (the METIS
import path, graph.py:232-256), so no partitioner runs.  Features are
uniform [0, 1) (cli.py:160); weights U(-0.5, 0.5), bias U(-0.1, 0.1)
(engine.py:418-420); grids are calibrated on batch 0 (cli.py:209).

``planted_batches`` builds each batch directly from its parts' local edges on
the GPU (equivalent to ``build_batch`` on the planted graph, checked by
tests/test_synth.py) so the 2.4M-node config does not need a global edge sort.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .bitpack import COLUMN_WISE, ROW_WISE, BitPlaneStack, PackedBitMatrix, pad8, pad128
from .engine import calibrate_model, gcn_model, gin_model
from .graph import SubgraphBatch
from .quantize import QuantParams, quantize_pack_device


@dataclass(frozen=True)
class GraphConfig:
    name: str
    model: str            # "gcn" | "gin"
    num_nodes: int
    num_edges: int        # undirected
    num_parts: int
    parts_per_batch: int
    in_dim: int
    hidden: int
    classes: int
    layers: int
    bits: int             # feature/activation bits
    wbits: int            # weight bits
    intra: float = 0.8


CONFIGS = {
    # configs[0]: the reference's CPU-runnable case
    "C1": GraphConfig("C1-gcn-3k", "gcn", 3000, 30000, 8, 8, 32, 16, 10, 2, 2, 2),
    # configs[1]: BlogCatalog-shaped, 16 planted parts in one batch, bit sweep 1..8
    "C2": GraphConfig("C2-gin-blogcatalog-10k", "gin", 10000, 334000, 16, 16, 128, 64, 39, 3, 4, 4),
    # configs[2]: ogbn-arxiv-shaped, 1500 METIS-style parts, 8 per batch
    "C3": GraphConfig("C3-gcn-arxiv-169k", "gcn", 169343, 1166243, 1500, 8, 128, 128, 40, 2, 4, 4),
    # configs[3]: ogbn-products-shaped, 1500 parts, 8 per batch
    "C4": GraphConfig("C4-gin-products-2.4M", "gin", 2449029, 61859140, 1500, 8, 100, 256, 47, 3, 8, 8),
}


def with_bits(cfg: GraphConfig, bits: int) -> GraphConfig:
    return GraphConfig(**{**cfg.__dict__, "bits": bits, "wbits": bits})


def part_bounds(cfg: GraphConfig) -> np.ndarray:
    return np.linspace(0, cfg.num_nodes, cfg.num_parts + 1).astype(np.int64)


def intra_edges_per_part(cfg: GraphConfig, bounds: np.ndarray) -> np.ndarray:
    """Undirected intra-part edge budget per part, proportional to size^2."""
    sizes = np.diff(bounds).astype(np.float64)
    w = sizes * sizes
    return np.floor(cfg.intra * cfg.num_edges * w / w.sum()).astype(np.int64)


def _part_local_edges(rng, size: int, m: int):
    s = rng.integers(0, size, m)
    d = rng.integers(0, size, m)
    return s, d


def planted_batches(cfg: GraphConfig, seed: int = 0, batch_ids=None, features_dtype=np.float32):
    """Build SubgraphBatches of the planted graph on the GPU.

    Returns (batches, features_per_batch_host, x_params).  Node ids are
    contiguous per part (part p owns [bounds[p], bounds[p+1])), parts are
    batched in order, ``parts_per_batch`` at a time (cli.py:179-186).
    """
    bounds = part_bounds(cfg)
    budget = intra_edges_per_part(cfg, bounds)
    n_batches = -(-cfg.num_parts // cfg.parts_per_batch)
    ids = range(n_batches) if batch_ids is None else batch_ids
    x_params = QuantParams(0.0, 1.0, cfg.bits)   # features U[0,1): grid [min, max) ~ [0, 1)
    batches, feats = [], []
    dev = N.device()
    for b in ids:
        rng = np.random.default_rng((seed, b))
        p0, p1 = b * cfg.parts_per_batch, min((b + 1) * cfg.parts_per_batch, cfg.num_parts)
        lo, hi = int(bounds[p0]), int(bounds[p1])
        total = hi - lo
        srcs, dsts = [], []
        for p in range(p0, p1):
            size = int(bounds[p + 1] - bounds[p])
            s, d = _part_local_edges(rng, size, int(budget[p]))
            off = int(bounds[p]) - lo
            srcs += [s + off, d + off]          # symmetrised (both directions)
            dsts += [d + off, s + off]
        diag = np.arange(total)
        src = N.to_device(np.concatenate(srcs + [diag]).astype(np.int64))
        dst = N.to_device(np.concatenate(dsts + [diag]).astype(np.int64))
        pr, pc = pad8(total), pad128(total)
        words = torch.zeros(pr * pc // 32, dtype=torch.int32, device=dev)
        N.call("qg_edges_to_bits", N.ptr(src), N.ptr(dst), src.numel(), total, N.ptr(words), pr, pc, N.stream())
        adj = PackedBitMatrix(COLUMN_WISE, total, total, pr, pc, words)
        x = rng.uniform(0.0, 1.0, (total, cfg.in_dim)).astype(features_dtype)
        r = quantize_pack_device(x, x_params, N.ROW_WISE_ID, 8, row_sums=True)
        fst = BitPlaneStack._wrap(ROW_WISE, total, cfg.in_dim, r["pr"], r["pc"], r["planes"])
        boundaries = bounds[p0:p1 + 1] - lo
        batches.append(SubgraphBatch(node_ids=np.arange(lo, hi), adjacency=adj, features=fst,
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


def batch_part_sizes(cfg: GraphConfig) -> list:
    """Node count of every part, per batch (parts batched in order, cli.py:179-186) --
    host-only, so ranks can plan the shard assignment before building anything."""
    sizes = np.diff(part_bounds(cfg))
    n_batches = -(-cfg.num_parts // cfg.parts_per_batch)
    return [sizes[b * cfg.parts_per_batch:(b + 1) * cfg.parts_per_batch] for b in range(n_batches)]
