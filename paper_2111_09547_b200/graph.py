"""Graph IO, partitioning, block-diagonal subgraph batches and their
single-transfer compound buffer (mirror of graph.py).

Graph IO (graph.py:85-156) and partition import/export (graph.py:232-262) are
host file formats, kept here with the reference's formats and error messages.
The balanced BFS partitioner (graph.py:190-229) runs natively
(``qg_partition_bfs``, csrc/qgtc_partition.cu): same assignment for the same
seed, O(E log E) instead of the reference's per-step frontier scan.

Batch construction runs on the GPU: kept intra-part edges are written
straight into packed adjacency words (``qg_edges_to_bits``; no dense
total x total matrix), features go through the fused bit_qnt kernel.
``unpack_batch`` moves a whole QGTB compound buffer with ONE host-to-device
copy and carves device views out of it.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .bitpack import (COLUMN_WISE, ROW_WISE, BitPlaneStack, PackedBitMatrix, _HEADER as _STACK_HEADER,
                      pad8, pad128, serialize)
from .errors import FormatError
from .quantize import QuantParams, quantize_pack_device

BUFFER_MAGIC = b"QGTB"
_BUFFER_HEADER = struct.Struct("<4sHIIBddBQQ")
GRAPH_MAGIC = b"QGTG"
_GRAPH_HEADER = struct.Struct("<4sHIQ")
BALANCE_SLACK = 0.10


@dataclass(eq=False)
class Graph:
    """Directed edge set over ``num_nodes`` nodes, duplicates collapsed (graph.py:48-82)."""

    num_nodes: int
    edges: np.ndarray
    features: np.ndarray | None = None

    def __post_init__(self):
        e = np.asarray(self.edges, dtype=np.int64).reshape(-1, 2)
        if e.size:
            if e.min() < 0 or e.max() >= self.num_nodes:
                raise ValueError("edge endpoint out of range")
            e = np.unique(e, axis=0)
        self.edges = e
        if self.features is not None:
            self.features = np.asarray(self.features, dtype=np.float64)
            if self.features.shape[0] != self.num_nodes:
                raise ValueError("feature row count must equal num_nodes")
        self._dev_edges = None

    @property
    def num_edges(self) -> int:
        return len(self.edges)

    def edge_set(self) -> set[tuple[int, int]]:
        """Edges as a Python set of (src, dst) pairs (graph.py:70-71)."""
        return set(map(tuple, self.edges.tolist()))

    def neighbors(self) -> list[list[int]]:
        """Undirected adjacency lists, sorted, no self references (graph.py:73-81)."""
        e = self.edges[self.edges[:, 0] != self.edges[:, 1]] if len(self.edges) else self.edges.reshape(0, 2)
        both = np.unique(np.concatenate([e, e[:, ::-1]]), axis=0)
        starts = np.searchsorted(both[:, 0], np.arange(self.num_nodes + 1))
        return [both[starts[v]:starts[v + 1], 1].tolist() for v in range(self.num_nodes)]

    def device_edges(self) -> torch.Tensor:
        if self._dev_edges is None:
            self._dev_edges = N.to_device(self.edges)
        return self._dev_edges


@dataclass(eq=False)
class PartitionAssignment:
    """Node -> part map (graph.py:159-175); members served from a cached CSR."""

    num_parts: int
    part_of: np.ndarray
    edge_cut: int | None = None

    def __post_init__(self):
        self.part_of = np.asarray(self.part_of, dtype=np.int64)
        if self.part_of.size and (self.part_of.min() < 0 or self.part_of.max() >= self.num_parts):
            raise ValueError("part index out of range")
        self._csr = None

    def members(self, part: int) -> np.ndarray:
        if self._csr is None:
            order = np.argsort(self.part_of, kind="stable")
            starts = np.searchsorted(self.part_of[order], np.arange(self.num_parts + 1))
            self._csr = (order, starts)
        order, starts = self._csr
        return order[starts[part]:starts[part + 1]]


# ------------------------------------------------------------------ graph IO
def load_graph(path, fmt: str = "edge-list-text") -> Graph:
    """Read a graph (graph.py:85-92): text lines ``src dst`` with an optional
    ``# nodes N`` header, or the binary QGTG image."""
    readers = {"edge-list-text": _read_text_graph, "binary": _read_binary_graph}
    if fmt not in readers:
        raise ValueError(f"unknown graph format {fmt!r}")
    return readers[fmt](path)


def _read_text_graph(path) -> Graph:
    # formats and messages of graph.py:95-125; a header bounds only the lines after it
    declared = None
    src, dst = [], []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            tok = raw.split()
            if not tok:
                continue
            if tok[0].startswith("#"):
                head = raw.strip()[1:].split()
                if len(head) != 2 or head[0] != "nodes" or not head[1].isdigit():
                    raise FormatError(f"{path}:{lineno}: unrecognized header {raw.strip()!r}")
                declared = int(head[1])
                continue
            if len(tok) != 2:
                raise FormatError(f"{path}:{lineno}: expected 'src dst', got {raw.strip()!r}")
            try:
                a, b = int(tok[0]), int(tok[1])
            except ValueError:
                raise FormatError(f"{path}:{lineno}: non-integer endpoint") from None
            if min(a, b) < 0:
                raise FormatError(f"{path}:{lineno}: negative node index")
            if declared is not None and max(a, b) >= declared:
                raise FormatError(f"{path}:{lineno}: index exceeds declared node count {declared}")
            src.append(a)
            dst.append(b)
    edges = np.stack([np.asarray(src, dtype=np.int64), np.asarray(dst, dtype=np.int64)], axis=1)
    n = declared if declared is not None else (int(edges.max()) + 1 if len(edges) else 0)
    return Graph(num_nodes=n, edges=edges)


def _read_binary_graph(path) -> Graph:
    data = open(path, "rb").read()
    if len(data) < _GRAPH_HEADER.size:
        raise FormatError("graph payload shorter than header")
    magic, version, n, m = _GRAPH_HEADER.unpack_from(data)
    if magic != GRAPH_MAGIC:
        raise FormatError(f"bad graph magic {magic!r}")
    if version != 1:
        raise FormatError(f"unsupported graph version {version}")
    if len(data) != _GRAPH_HEADER.size + 8 * m:
        raise FormatError(f"graph payload length {len(data)} != expected {_GRAPH_HEADER.size + 8 * m}")
    pairs = np.frombuffer(data, dtype="<u4", count=2 * m, offset=_GRAPH_HEADER.size)
    return Graph(num_nodes=n, edges=pairs.astype(np.int64).reshape(-1, 2))


def save_graph(g: Graph, path, fmt: str = "edge-list-text") -> None:
    """Write a graph in either format (graph.py:128-141)."""
    if fmt == "edge-list-text":
        body = "\n".join(f"{a} {b}" for a, b in g.edges.tolist())
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(f"# nodes {g.num_nodes}\n" + (body + "\n" if body else ""))
    elif fmt == "binary":
        with open(path, "wb") as fh:
            fh.write(_GRAPH_HEADER.pack(GRAPH_MAGIC, 1, g.num_nodes, g.num_edges))
            fh.write(np.ascontiguousarray(g.edges, dtype="<u4").tobytes())
    else:
        raise ValueError(f"unknown graph format {fmt!r}")


# ------------------------------------------------------------- partitioning
def edge_cut(g: Graph, assign: PartitionAssignment) -> int:
    """Distinct undirected edges whose endpoints sit in different parts (graph.py:178-187)."""
    if not len(g.edges):
        return 0
    lo, hi = g.edges.min(axis=1), g.edges.max(axis=1)
    und = np.unique(lo * np.int64(g.num_nodes) + hi)
    a, b = und // g.num_nodes, und % g.num_nodes
    return int(np.count_nonzero(assign.part_of[a] != assign.part_of[b]))


def partition(g: Graph, num_parts: int, seed: int = 0) -> PartitionAssignment:
    """Balanced BFS-grown greedy partition (graph.py:190-229) on the native host
    partitioner: identical part_of to the reference for the same seed."""
    n = g.num_nodes
    if not 1 <= num_parts <= n:
        raise ValueError(f"num_parts must be in [1, {n}], got {num_parts}")
    e = g.edges[g.edges[:, 0] != g.edges[:, 1]] if len(g.edges) else g.edges.reshape(0, 2)
    both = np.unique(np.concatenate([e, e[:, ::-1]]), axis=0) if len(e) else e
    indptr = np.searchsorted(both[:, 0], np.arange(n + 1)).astype(np.int64)
    nbrs = np.ascontiguousarray(both[:, 1], dtype=np.int64)
    part_of = np.empty(n, dtype=np.int64)
    rc = N.lib().qg_partition_bfs(n, indptr.ctypes.data, nbrs.ctypes.data if len(nbrs) else None,
                                  int(num_parts), int(seed), part_of.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"qg_partition_bfs failed ({rc})")
    assign = PartitionAssignment(num_parts=num_parts, part_of=part_of)
    assign.edge_cut = edge_cut(g, assign)
    return assign


def import_partition(path, num_nodes: int | None = None, num_parts: int | None = None) -> PartitionAssignment:
    """One part index per line, e.g. METIS output (graph.py:232-256)."""
    parts = []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            t = raw.strip()
            if t:
                try:
                    parts.append(int(t))
                except ValueError:
                    raise FormatError(f"{path}:{lineno}: not an integer") from None
    if num_nodes is not None and len(parts) != num_nodes:
        raise ValueError(f"expected {num_nodes} lines, found {len(parts)}")
    if not parts:
        raise ValueError("empty partition file")
    arr = np.asarray(parts, dtype=np.int64)
    if arr.min() < 0:
        raise ValueError("negative part index")
    count = int(arr.max()) + 1
    if num_parts is not None:
        if count > num_parts:
            raise ValueError(f"part index {count - 1} >= num_parts {num_parts}")
        count = num_parts
    return PartitionAssignment(num_parts=count, part_of=arr)


def export_partition(assign: PartitionAssignment, path) -> None:
    """Inverse of import_partition (graph.py:259-262)."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("".join(f"{p}\n" for p in assign.part_of.tolist()))


class SubgraphBatch:
    """Block-diagonal binarized adjacency + quantized features (graph.py:265-305).

    ``node_ids`` / ``boundaries`` are host metadata; adjacency and features are
    device-resident.  ``degrees()`` comes from the cached tile scan.
    """

    def __init__(self, node_ids, adjacency: PackedBitMatrix, features: BitPlaneStack | None, boundaries,
                 x_params: QuantParams | None = None, feat_row_sums: torch.Tensor | None = None):
        self.node_ids = np.asarray(node_ids, dtype=np.int64)
        self.boundaries = np.asarray(boundaries, dtype=np.int64)
        self.adjacency = adjacency
        self.features = features
        self.x_params = x_params
        self._feat_row_sums = feat_row_sums
        total = len(self.node_ids)
        if self.boundaries[0] != 0 or self.boundaries[-1] != total:
            raise ValueError("boundaries must start at 0 and end at total nodes")
        if adjacency.logical_rows != total or adjacency.logical_cols != total:
            raise ValueError("adjacency must be square over the batch nodes")

    @property
    def total_nodes(self) -> int:
        return len(self.node_ids)

    @property
    def num_subgraphs(self) -> int:
        return len(self.boundaries) - 1

    def degrees(self) -> np.ndarray:
        """Out-degree per batch row from the packed adjacency, int64 (graph.py:292-295)."""
        from .bitgemm import _schedule
        return _schedule(self.adjacency).degrees.cpu().numpy()

    def __eq__(self, other):
        return (isinstance(other, SubgraphBatch) and np.array_equal(self.node_ids, other.node_ids)
                and np.array_equal(self.boundaries, other.boundaries) and self.adjacency == other.adjacency
                and self.features == other.features and self.x_params == other.x_params)

    __hash__ = None


def _local_edges(g: Graph, assign: PartitionAssignment, groups, node_ids: np.ndarray):
    """Kept (intra-part) edges in batch-local indices, on the device (graph.py:328-338)."""
    dev = N.device()
    e = g.device_edges()
    if e.numel() == 0:
        z = torch.zeros(0, dtype=torch.int64, device=dev)
        return z, z
    local = torch.full((g.num_nodes,), -1, dtype=torch.int64, device=dev)
    local[N.to_device(node_ids)] = torch.arange(len(node_ids), device=dev)
    block_of = torch.full((g.num_nodes,), -1, dtype=torch.int64, device=dev)
    for b, gr in enumerate(groups):
        block_of[N.to_device(gr)] = b
    s, d = e[:, 0], e[:, 1]
    keep = (block_of[s] >= 0) & (block_of[s] == block_of[d])
    return local[s[keep]], local[d[keep]]


def build_batch(g: Graph, assign: PartitionAssignment, part_ids, x_quant: QuantParams | None = None, *,
                add_self_loops: bool = True) -> SubgraphBatch:
    """Induced block-diagonal batch for ``part_ids`` (graph.py:308-357), built on the GPU."""
    part_ids = list(part_ids)
    if len(part_ids) != len(set(part_ids)):
        raise ValueError("part_ids must be distinct")
    groups = [assign.members(p) for p in part_ids]
    node_ids = np.concatenate(groups) if groups else np.zeros(0, dtype=np.int64)
    total = len(node_ids)
    if total == 0:
        raise ValueError("empty batch")
    boundaries = np.cumsum([0] + [len(gr) for gr in groups])
    src, dst = _local_edges(g, assign, groups, node_ids)
    if add_self_loops:
        diag = torch.arange(total, device=src.device, dtype=torch.int64)
        src, dst = torch.cat([src, diag]), torch.cat([dst, diag])
    pr, pc = pad8(total), pad128(total)
    words = torch.zeros(pr * pc // 32, dtype=torch.int32, device=src.device)
    N.call("qg_edges_to_bits", N.ptr(src.contiguous()), N.ptr(dst.contiguous()), src.numel(), total,
           N.ptr(words), pr, pc, N.stream())
    adjacency = PackedBitMatrix(COLUMN_WISE, total, total, pr, pc, words)
    features, row_sums = None, None
    if g.features is not None:
        if x_quant is None:
            raise ValueError("x_quant is required to quantize node features")
        r = quantize_pack_device(g.features[node_ids], x_quant, N.ROW_WISE_ID, 8, row_sums=True)
        features = BitPlaneStack._wrap(ROW_WISE, r["rows"], r["cols"], r["pr"], r["pc"], r["planes"])
        row_sums = r["row_sums"]
    return SubgraphBatch(node_ids=node_ids, adjacency=adjacency, features=features, boundaries=boundaries,
                         x_params=x_quant, feat_row_sums=row_sums)


@dataclass(eq=False)
class CompoundBuffer:
    """One contiguous byte image of a batch (graph.py:360-371)."""

    data: bytes

    @property
    def nbytes(self) -> int:
        return len(self.data)

    def __eq__(self, other):
        return isinstance(other, CompoundBuffer) and self.data == other.data


def pack_batch(b: SubgraphBatch) -> CompoundBuffer:
    """Serialize a batch into one transfer object, byte-identical to graph.py:374-397."""
    adj_stack = BitPlaneStack._wrap(COLUMN_WISE, *b.adjacency.dims(), b.adjacency.dwords.reshape(1, -1))
    adj_bytes = serialize(adj_stack)
    feat_bytes = serialize(b.features) if b.features is not None else b""
    ns, total = b.num_subgraphs, b.total_nodes
    fixed = _BUFFER_HEADER.size + 4 * (ns + 1) + 4 * total
    adj_off = fixed
    feat_off = adj_off + len(adj_bytes) if feat_bytes else 0
    if b.x_params is not None:
        amin, amax, bits = b.x_params.alpha_min, b.x_params.alpha_max, b.x_params.bits
    else:
        amin, amax, bits = 0.0, 0.0, 0
    fbits = b.features.bits if b.features is not None else 0
    header = _BUFFER_HEADER.pack(BUFFER_MAGIC, 1, ns, total, fbits, amin, amax, bits, adj_off, feat_off)
    body = (header + b.boundaries.astype("<u4").tobytes() + b.node_ids.astype("<u4").tobytes()
            + adj_bytes + feat_bytes)
    return CompoundBuffer(data=body)


def _parse_stack_header(data, off, end):
    if end - off < _STACK_HEADER.size:
        raise FormatError("payload shorter than header")
    return _STACK_HEADER.unpack_from(data, off)


def unpack_batch(buf, *, pinned: bool = False) -> SubgraphBatch:
    """Inverse of pack_batch (graph.py:400-431): ONE host-to-device copy of the buffer.

    The header is validated on the host; adjacency and feature words become
    device views into the transferred buffer (re-aligned to 16 B on device
    when the section offset is not, since the GEMM kernels use 128-bit loads).
    """
    data = buf.data if isinstance(buf, CompoundBuffer) else bytes(buf)
    if len(data) < _BUFFER_HEADER.size:
        raise FormatError("compound buffer shorter than header")
    magic, version, ns, total, fbits, amin, amax, bits, adj_off, feat_off = _BUFFER_HEADER.unpack_from(data)
    if magic != BUFFER_MAGIC:
        raise FormatError(f"bad compound-buffer magic {magic!r}")
    if version != 1:
        raise FormatError(f"unsupported compound-buffer version {version}")
    off = _BUFFER_HEADER.size
    need = off + 4 * (ns + 1) + 4 * total
    if len(data) < need or adj_off != need:
        raise FormatError("corrupt compound-buffer header")
    boundaries = np.frombuffer(data, dtype="<u4", count=ns + 1, offset=off).astype(np.int64)
    node_ids = np.frombuffer(data, dtype="<u4", count=total, offset=off + 4 * (ns + 1)).astype(np.int64)
    adj_end = feat_off if feat_off else len(data)
    sections = [(adj_off, adj_end)] + ([(feat_off, len(data))] if feat_off else [])
    metas = []
    for (s0, s1) in sections:
        magic2, ver2, orient, sbits, lr, lc, pr, pc = _parse_stack_header(data, s0, s1)
        if magic2 != b"QGTC":
            raise FormatError(f"bad magic {magic2!r}")
        if ver2 != 1:
            raise FormatError(f"unsupported version {ver2}")
        if orient not in (0, 1):
            raise FormatError(f"bad orientation byte {orient}")
        if not 1 <= sbits <= 64:
            raise FormatError(f"bad plane count {sbits}")
        if s1 - s0 != _STACK_HEADER.size + sbits * (pr * pc // 32) * 4:
            raise FormatError(f"payload length {s1 - s0} != expected "
                              f"{_STACK_HEADER.size + sbits * (pr * pc // 32) * 4}")
        metas.append((orient, sbits, lr, lc, pr, pc))
    if metas[0][1] != 1:
        raise FormatError("adjacency section must be a 1-bit stack")
    if feat_off and metas[1][1] != fbits:
        raise FormatError("feature bit count disagrees with header")
    host = torch.frombuffer(bytearray(data), dtype=torch.uint8)
    if pinned:
        host = host.pin_memory()
    dev_buf = host.to(N.device(), non_blocking=pinned)          # the single H2D transfer
    stacks = []
    for (s0, _), (orient, sbits, lr, lc, pr, pc) in zip(sections, metas):
        w0 = s0 + _STACK_HEADER.size
        nbytes = sbits * (pr * pc // 32) * 4
        view = dev_buf[w0:w0 + nbytes]
        if w0 % 16:
            view = view.clone()
        words = view.view(torch.int32).reshape(sbits, -1)
        stacks.append(BitPlaneStack._wrap(COLUMN_WISE if orient == 0 else ROW_WISE, lr, lc, pr, pc, words))
    params = QuantParams(amin, amax, bits) if fbits else None
    return SubgraphBatch(node_ids=node_ids, adjacency=stacks[0].planes[0],
                         features=stacks[1] if feat_off else None, boundaries=boundaries, x_params=params)


def float32_dense_bytes(b: SubgraphBatch) -> int:
    """Size of the naive float32 dense encoding of the same batch (graph.py:434-440)."""
    n = b.total_nodes
    size = 4 * n * n
    if b.features is not None:
        size += 4 * n * b.features.logical_cols
    return size


# ---------------------------------------------------------------- QGT2 wire
# Bandwidth/alignment-optimised compound format for the device fast path
# (SURVEY.md section 8(f) rank 1).  Same content as QGTB, but every section
# starts on a 256-byte boundary so device views are 128-bit loadable.
#   header (64 B): magic "QGT2", u16 version, u16 flags, u32 num_subgraphs,
#   u32 total_nodes, u8 feature_bits, u8 x_bits, u16 reserved, f64 amin,
#   f64 amax, u32 adj_pr, u32 adj_pc, u32 feat_pr, u32 feat_pc, u32 in_dim
#   then sections: boundaries u32[ns+1], node_ids u32[total], adjacency
#   words, feature plane words.
V2_MAGIC = b"QGT2"
_V2_HEADER = struct.Struct("<4sHHIIBBHddIIIII")
_V2_ALIGN = 256


def _v2_layout(ns: int, total: int, adj_words: int, feat_words: int):
    def up(x):
        return -(-x // _V2_ALIGN) * _V2_ALIGN
    o_b = up(_V2_HEADER.size)
    o_ids = up(o_b + 4 * (ns + 1))
    o_adj = up(o_ids + 4 * total)
    o_feat = up(o_adj + 4 * adj_words)
    end = up(o_feat + 4 * feat_words)
    return o_b, o_ids, o_adj, o_feat, end


def pack_batch_v2(b: SubgraphBatch) -> bytes:
    """QGT2 image of a batch (row-wise feature planes, column-wise adjacency)."""
    a, f = b.adjacency, b.features
    fw = 0 if f is None else int(f.dwords.numel())
    ns, total = b.num_subgraphs, b.total_nodes
    o_b, o_ids, o_adj, o_feat, end = _v2_layout(ns, total, int(a.dwords.numel()), fw)
    out = bytearray(end)
    xp = b.x_params
    _V2_HEADER.pack_into(out, 0, V2_MAGIC, 1, 0, ns, total, 0 if f is None else f.bits,
                         0 if xp is None else xp.bits, 0, 0.0 if xp is None else xp.alpha_min,
                         0.0 if xp is None else xp.alpha_max, a.padded_rows, a.padded_cols,
                         0 if f is None else f.padded_rows, 0 if f is None else f.padded_cols,
                         0 if f is None else f.logical_cols)
    out[o_b:o_b + 4 * (ns + 1)] = b.boundaries.astype("<u4").tobytes()
    out[o_ids:o_ids + 4 * total] = b.node_ids.astype("<u4").tobytes()
    out[o_adj:o_adj + 4 * a.dwords.numel()] = a.dwords.cpu().numpy().astype("<i4").tobytes()
    if f is not None:
        out[o_feat:o_feat + 4 * fw] = f.dwords.cpu().numpy().astype("<i4").tobytes()
    return bytes(out)


def batch_from_v2(header_bytes: bytes, dev_buf: torch.Tensor, base: int = 0) -> SubgraphBatch:
    """Device views of a QGT2 image already resident at ``dev_buf[base:]``.

    Only the header / id sections are read on the host (from ``header_bytes``);
    the adjacency and feature words are zero-copy views into the device buffer.
    """
    (magic, version, _flags, ns, total, fbits, xbits, _r, amin, amax, apr, apc, fpr, fpc,
     in_dim) = _V2_HEADER.unpack_from(header_bytes)
    if magic != V2_MAGIC:
        raise FormatError(f"bad compound-buffer magic {magic!r}")
    if version != 1:
        raise FormatError(f"unsupported compound-buffer version {version}")
    fw = fbits * fpr * fpc // 32
    o_b, o_ids, o_adj, o_feat, end = _v2_layout(ns, total, apr * apc // 32, fw)
    if len(header_bytes) < o_adj:
        raise FormatError("compound buffer shorter than its id sections")
    boundaries = np.frombuffer(header_bytes, dtype="<u4", count=ns + 1, offset=o_b).astype(np.int64)
    node_ids = np.frombuffer(header_bytes, dtype="<u4", count=total, offset=o_ids).astype(np.int64)
    if (base + o_adj) % 16:
        raise FormatError("QGT2 image must start 16-byte aligned")
    adj_w = dev_buf[base + o_adj: base + o_adj + 4 * (apr * apc // 32)].view(torch.int32)
    adj = PackedBitMatrix(COLUMN_WISE, total, total, apr, apc, adj_w)
    feats = None
    params = None
    if fbits:
        fwords = dev_buf[base + o_feat: base + o_feat + 4 * fw].view(torch.int32).reshape(fbits, -1)
        feats = BitPlaneStack._wrap(ROW_WISE, total, in_dim, fpr, fpc, fwords)
        params = QuantParams(amin, amax, xbits)
    return SubgraphBatch(node_ids=node_ids, adjacency=adj, features=feats, boundaries=boundaries,
                         x_params=params)


# ------------------------------------------------------- QGT3 tile-sparse wire
# QGT2 ships the dense packed adjacency (pad8(n) x pad128(n) bits) although a
# block-diagonal batch has mostly all-zero 8x128 tiles (C2: ~92%).  QGT3 ships the
# zero-tile-jumping schedule and ONLY the non-zero 128x128 bit blocks (2 KB each,
# 128 rows x 4 words, the device `packed` layout of tiled.BlockedAdjacency), so the
# single H2D carries ~8x fewer bytes and the device expands the blocks straight
# into the tensor-core operand layout (qg_block_prepare, no gather).
#   header (96 B): magic "QGT3", u16 version, u16 flags, u32 num_subgraphs,
#   u32 total_nodes, u8 feature_bits, u8 x_bits, u16 reserved, f64 amin, f64 amax,
#   u32 adj_pr, u32 adj_pc, u32 feat_pr, u32 feat_pc, u32 in_dim, u32 n_row_blocks,
#   u32 n_blocks, u64 nonzero_8x128_tiles
#   sections (256-B aligned): boundaries u32[ns+1], node_ids u32[total],
#   blk_count i32[nrb], blk_base i32[nrb], blk_kt i32[nb], blk_rb i32[nb],
#   blocks u32[nb][128][4], feature plane words.
V3_MAGIC = b"QGT3"
_V3_HEADER = struct.Struct("<4sHHIIBBHddIIIIIIIQ")


def _v3_layout(ns: int, total: int, nrb: int, nb: int, feat_words: int):
    def up(x):
        return -(-x // _V2_ALIGN) * _V2_ALIGN
    o = [up(_V3_HEADER.size)]
    for size in (4 * (ns + 1), 4 * total, 4 * nrb, 4 * nrb, 4 * nb, 4 * nb, 2048 * nb, 4 * feat_words):
        o.append(up(o[-1] + size))
    return o        # boundaries, ids, count, base, kt, rb, blocks, feats, end


def pack_batch_v3(b: SubgraphBatch) -> bytes:
    """QGT3 image of a batch: schedule + non-zero 128x128 adjacency blocks + feature planes."""
    from .tiled import blocked
    a, f = b.adjacency, b.features
    blk = blocked(a)
    fw = 0 if f is None else int(f.dwords.numel())
    ns, total, nrb, nb = b.num_subgraphs, b.total_nodes, blk.nrb, blk.nblocks
    o = _v3_layout(ns, total, nrb, nb, fw)
    out = bytearray(o[-1])
    xp = b.x_params
    _V3_HEADER.pack_into(out, 0, V3_MAGIC, 1, 0, ns, total, 0 if f is None else f.bits,
                         0 if xp is None else xp.bits, 0, 0.0 if xp is None else xp.alpha_min,
                         0.0 if xp is None else xp.alpha_max, a.padded_rows, a.padded_cols,
                         0 if f is None else f.padded_rows, 0 if f is None else f.padded_cols,
                         0 if f is None else f.logical_cols, nrb, nb, int(blk.nz8))
    secs = [b.boundaries.astype("<u4"), b.node_ids.astype("<u4"),
            blk.blk_count.cpu().numpy().astype("<i4"), blk.blk_base.cpu().numpy().astype("<i4"),
            blk.blk_kt.cpu().numpy().astype("<i4"), blk.blk_rb.cpu().numpy().astype("<i4"),
            blk.packed[:nb].cpu().numpy().astype("<i4")]
    if f is not None:
        secs.append(f.dwords.cpu().numpy().astype("<i4"))
    for off, arr in zip(o, secs):
        raw = arr.tobytes()
        out[off:off + len(raw)] = raw
    return bytes(out)


def v3_feature_offset(image: bytes) -> int:
    """Byte offset of the feature-plane section inside a QGT3 image (the last section)."""
    (_m, _v, _f, ns, total, fbits, _x, _r, _a, _b, _apr, _apc, fpr, fpc, _d, nrb, nb,
     _nz) = _V3_HEADER.unpack_from(image)
    return _v3_layout(ns, total, nrb, nb, fbits * fpr * fpc // 32)[7]


class BlockSparseAdjacency(PackedBitMatrix):
    """Column-wise 1-bit adjacency known only by its non-zero 128x128 blocks (QGT3).

    The engine reads the blocks directly; the dense ``words`` (the reference's
    layout) are scattered from them on first access, for API parity."""

    def __init__(self, total, pr, pc, blocked_adj):
        self.orientation = COLUMN_WISE
        self.logical_rows = self.logical_cols = int(total)
        self.padded_rows, self.padded_cols = int(pr), int(pc)
        self._tilemap = None
        self._schedule = None
        self._np = None
        self._dense = None
        self._blocked = blocked_adj

    @property
    def dwords(self) -> torch.Tensor:
        if self._dense is None:
            blk = self._blocked
            pr, pc = self.padded_rows, self.padded_cols
            rows128 = -(-pr // 128) * 128
            dense = torch.zeros((rows128, pc // 32), dtype=torch.int32, device=blk.packed.device)
            if blk.nblocks:
                view = dense.view(rows128 // 128, 128, pc // 128, 4)
                view[blk.blk_rb.long(), :, blk.blk_kt.long(), :] = blk.packed[:blk.nblocks]
            self._dense = dense[:pr].reshape(-1)
        return self._dense

    @dwords.setter
    def dwords(self, value):
        self._dense = value


def batch_from_v3(header_bytes: bytes, dev_buf: torch.Tensor, base: int = 0) -> SubgraphBatch:
    """Device views of a QGT3 image resident at ``dev_buf[base:]``; blocks are expanded by
    ``BlockedAdjacency.refresh()`` (the epoch graph does it every step)."""
    from .tiled import BlockedAdjacency
    (magic, version, _flags, ns, total, fbits, xbits, _r, amin, amax, apr, apc, fpr, fpc, in_dim, nrb, nb,
     nz8) = _V3_HEADER.unpack_from(header_bytes)
    if magic != V3_MAGIC:
        raise FormatError(f"bad compound-buffer magic {magic!r}")
    if version != 1:
        raise FormatError(f"unsupported compound-buffer version {version}")
    fw = fbits * fpr * fpc // 32
    o = _v3_layout(ns, total, nrb, nb, fw)
    if len(header_bytes) < o[2]:
        raise FormatError("compound buffer shorter than its id sections")
    if (base + o[2]) % 256:
        raise FormatError("QGT3 image must start 256-byte aligned")
    boundaries = np.frombuffer(header_bytes, dtype="<u4", count=ns + 1, offset=o[0]).astype(np.int64)
    node_ids = np.frombuffer(header_bytes, dtype="<u4", count=total, offset=o[1]).astype(np.int64)

    def view(k, count, dtype=torch.int32):
        return dev_buf[base + o[k]: base + o[k] + 4 * count].view(dtype)

    blk = BlockedAdjacency.from_blocks(total, apr, view(2, nrb), view(3, nrb), view(4, nb), view(5, nb),
                                       view(6, nb * 512).view(max(nb, 0), 128, 4), nb, nz8)
    adj = BlockSparseAdjacency(total, apr, apc, blk)
    blk._src = adj
    feats = params = None
    if fbits:
        feats = BitPlaneStack._wrap(ROW_WISE, total, in_dim, fpr, fpc, view(7, fw).reshape(fbits, -1))
        params = QuantParams(amin, amax, xbits)
    return SubgraphBatch(node_ids=node_ids, adjacency=adj, features=feats, boundaries=boundaries,
                         x_params=params)
