"""Host-only (numpy) half of the synthetic workloads -- no torch, no native library.

The planted-partition generator of SURVEY.md section 8(d), shared by the GPU
path (``synth.planted_batches``) and the reference CPU arm (``bench.py --impl
reference``, which must build its inputs without this package's kernels).  For
batch ``b`` one ``np.random.default_rng((seed, b))`` stream yields, in order,
every part's local edge endpoints (src then dst, ``budget[p]`` each) and then
the batch's U[0, 1) features (cli.py:160), so both sides see identical inputs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


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


def batch_part_sizes(cfg: GraphConfig) -> list:
    """Node count of every part, per batch (parts batched in order, cli.py:179-186) --
    host-only, so ranks can plan the shard assignment before building anything."""
    sizes = np.diff(part_bounds(cfg))
    n_batches = -(-cfg.num_parts // cfg.parts_per_batch)
    return [sizes[b * cfg.parts_per_batch:(b + 1) * cfg.parts_per_batch] for b in range(n_batches)]


def num_batches(cfg: GraphConfig) -> int:
    return -(-cfg.num_parts // cfg.parts_per_batch)


def host_batch(cfg: GraphConfig, seed: int, b: int, features_dtype=np.float32):
    """Batch ``b`` of the planted graph on the host.

    Returns ``(local_edges, boundaries, features)``: ``local_edges`` = one
    (src, dst) pair of int64 arrays per part, endpoints local to the PART (not yet
    symmetrised, no self loops); ``boundaries`` = batch-local part offsets
    (len parts + 1); ``features`` = (total, in_dim) U[0, 1) values."""
    bounds = part_bounds(cfg)
    budget = intra_edges_per_part(cfg, bounds)
    rng = np.random.default_rng((seed, b))
    p0, p1 = b * cfg.parts_per_batch, min((b + 1) * cfg.parts_per_batch, cfg.num_parts)
    lo, hi = int(bounds[p0]), int(bounds[p1])
    edges = []
    for p in range(p0, p1):
        size = int(bounds[p + 1] - bounds[p])
        edges.append(_part_local_edges(rng, size, int(budget[p])))
    x = rng.uniform(0.0, 1.0, (hi - lo, cfg.in_dim)).astype(features_dtype)
    return edges, bounds[p0:p1 + 1] - lo, x


def batch_edge_list(edges, boundaries, self_loops: bool = True) -> np.ndarray:
    """(E, 2) batch-local directed edge list: every part's edges symmetrised (both
    directions) and offset to the batch, plus the diagonal -- the edge set whose
    induced block-diagonal batch is what graph.py:308-357 builds."""
    parts = []
    for (s, d), off in zip(edges, boundaries[:-1]):
        parts.append(np.stack([s + off, d + off], 1))
        parts.append(np.stack([d + off, s + off], 1))
    if self_loops:
        diag = np.arange(int(boundaries[-1]), dtype=np.int64)
        parts.append(np.stack([diag, diag], 1))
    return np.concatenate(parts).astype(np.int64)
