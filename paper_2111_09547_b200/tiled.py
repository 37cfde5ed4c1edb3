"""Tiled fast path: operands in the UMMA K-major layout + grouped multi-batch GEMMs.

The engine's hot loop (engine.py:235-332) runs here.  For every GEMM the left
and right operands are stored in HBM exactly as the tcgen05 MMA reads them from
shared memory (see include/qgtc_b200.h "tiled fast path"), so the kernel moves
each K tile with two bulk copies and never unpacks bits on the critical path:

* the 1-bit adjacency -> its non-zero 128x128 blocks as 0/1 bytes (16 KB each),
  built once per batch from the zero-tile schedule (the reference caches the
  scan on the operand, bitgemm.py:222-233) and reused by every layer;
* activations -> u8 code caches written by the producing epilogue in the
  layout their consumer reads (left-tiled for X.W, right-tiled for A.X);
* weights -> right-tiled codes of W, once per model.

A layer stage over ALL batches of an epoch is one ``qg_tiled_gemm`` launch
(one segment per batch), so the 188-batch configs launch 2 kernels per layer.
Packed planes (the reference's ``words``) are materialised lazily from the
code caches only when the API asks for them.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _native as N
from .bitpack import COLUMN_WISE, ROW_WISE, BitPlaneStack, pad128, padded_dims

TILE = 128


def npad_of(n: int) -> int:
    """Right-operand column padding: a power of two >= 32 up to 256, else a multiple of 256."""
    if n <= 256:
        p = 32
        while p < n:
            p *= 2
        return p
    return -(-n // 256) * 256


class TSeg(ctypes.Structure):
    """Mirror of ``qg_tseg``."""

    _fields_ = [("a", ctypes.c_void_p), ("b", ctypes.c_void_p), ("blk_count", ctypes.c_void_p),
                ("blk_base", ctypes.c_void_p), ("blk_kt", ctypes.c_void_p), ("row_sums", ctypes.c_void_p),
                ("q_codes", ctypes.c_void_p), ("q_row_sums", ctypes.c_void_p), ("out_real", ctypes.c_void_p),
                ("out_i32", ctypes.c_void_p), ("status", ctypes.c_void_p), ("m", ctypes.c_int64),
                ("r128", ctypes.c_int64), ("cta_begin", ctypes.c_int64), ("k_tiles", ctypes.c_int32),
                ("pad_", ctypes.c_int32), ("reserved0", ctypes.c_int64), ("tmap_a", ctypes.c_uint8 * 128),
                ("tmap_b", ctypes.c_uint8 * 128)]


class TiledArgs(ctypes.Structure):
    """Mirror of ``qg_tiled_args``."""

    _fields_ = [("segs", ctypes.c_void_p), ("nsegs", ctypes.c_int32), ("a_blocks", ctypes.c_int32),
                ("total_ctas", ctypes.c_int64), ("b_npad", ctypes.c_int64), ("n", ctypes.c_int64),
                ("bn", ctypes.c_int32), ("n_tiles", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("out_layout", ctypes.c_int32), ("out_npad", ctypes.c_int64),
                ("epi", ctypes.POINTER(N.Epilogue)), ("phase_ns", ctypes.c_void_p), ("a_bits", ctypes.c_int32),
                ("pair", ctypes.c_int32), ("chain", ctypes.c_void_p), ("reserved1", ctypes.c_void_p),
                ("reserved2", ctypes.c_void_p), ("reserved3", ctypes.c_int32), ("pad3_", ctypes.c_int32)]


class Chain(ctypes.Structure):
    """Mirror of ``qg_chain``: a dense stage-2 GEMM fused behind a tiled stage."""

    _fields_ = [("w", ctypes.c_void_p), ("w_npad", ctypes.c_int64), ("n", ctypes.c_int64),
                ("out_layout", ctypes.c_int32), ("reserved", ctypes.c_int32), ("out_npad", ctypes.c_int64),
                ("epi", ctypes.POINTER(N.Epilogue))]


_SIGS_DONE = False

# qg_tiled_gemm launches issued so far (runtime.EpochRunner counts those of its graph)
LAUNCHES = 0

# An event the first adjacency-block launch must wait on (the e2e runner's side-stream
# H2D of the schedule + blocks and their expansion); cleared once joined.
PENDING_JOIN = None

# 2-SM CTA pairs for large GEMM stages (QG_PAIR=0 disables)
PAIR = os.environ.get("QG_PAIR", "1") != "0"


def _lib():
    global _SIGS_DONE
    L = N.lib()
    if not _SIGS_DONE:
        L.qg_tiled_gemm.argtypes = [ctypes.POINTER(TiledArgs), ctypes.c_void_p]
        L.qg_tiled_gemm.restype = ctypes.c_int
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.qg_block_prepare.argtypes = [vp, i64, i64, i64, vp, vp, i64, vp, vp, vp, vp]
        L.qg_block_prepare.restype = ctypes.c_int
        L.qg_codes_to_tiles.argtypes = [vp, i64, i64, i64, i32, i64, vp, vp]
        L.qg_codes_to_tiles.restype = ctypes.c_int
        L.qg_tiles_to_codes.argtypes = [vp, i64, i64, i32, i64, vp, i64, vp]
        L.qg_tiles_to_codes.restype = ctypes.c_int
        L.qg_encode_linear_map.argtypes = [vp, i64, i32, vp]
        L.qg_encode_linear_map.restype = ctypes.c_int
        _SIGS_DONE = True
    return L


# ------------------------------------------------------------------ adjacency
class BlockedAdjacency:
    """Non-zero 128x128 blocks of a column-wise 1-bit adjacency, expanded to bytes."""

    def __init__(self, a, schedule):
        # host view of the zero-tile schedule (one sync, at build time)
        counts = schedule.blk_count.cpu().numpy().astype(np.int64)
        lists = schedule.blk_list.cpu().numpy()
        self.nrb = len(counts)
        base = np.zeros(self.nrb, dtype=np.int64)
        if self.nrb:
            base[1:] = np.cumsum(counts)[:-1]
        self.nblocks = int(counts.sum())
        rb_of = np.repeat(np.arange(self.nrb), counts)
        kt_of = np.concatenate([lists[r, :counts[r]] for r in range(self.nrb)]) if self.nblocks else \
            np.zeros(0, np.int64)
        dev = a.dwords.device
        self.blk_count = schedule.blk_count
        self.blk_base = torch.from_numpy(base.astype(np.int32)).to(dev)
        self.blk_kt = torch.from_numpy(kt_of.astype(np.int32)).to(dev)
        self.blk_rb = torch.from_numpy(rb_of.astype(np.int32)).to(dev)
        self.packed = torch.empty((max(self.nblocks, 1), 128, 4), dtype=torch.int32, device=dev)
        self._bytes = None
        self.degrees = torch.zeros(a.logical_rows, dtype=torch.int64, device=dev)
        self.m = a.logical_rows
        self.r128 = pad128(a.logical_rows)
        self._src = a
        # non-zero 8x128 tiles: the reference's unit of work (bitgemm.py:335-347)
        self.nz8 = schedule.rt * schedule.ct - schedule.zeros
        self.refresh()

    @classmethod
    def from_blocks(cls, rows, padded_rows, blk_count, blk_base, blk_kt, blk_rb, packed, nblocks, nz8):
        """Adopt a shipped schedule + packed blocks (QGT3 wire views); ``refresh()``
        expands them (no gather: the dense words never exist on the device)."""
        self = cls.__new__(cls)
        self.nrb = int(blk_count.numel())
        self.nblocks = int(nblocks)
        dev = blk_count.device
        self.blk_count, self.blk_base, self.blk_kt, self.blk_rb = blk_count, blk_base, blk_kt, blk_rb
        self.packed = packed if nblocks else torch.zeros((1, 128, 4), dtype=torch.int32, device=dev)
        self._bytes = None
        self.degrees = torch.zeros(int(rows), dtype=torch.int64, device=dev)
        self.m = int(rows)
        self.r128 = pad128(int(rows))
        self.nz8 = int(nz8)
        self._src = None
        self._gather = False
        self.refresh()
        return self

    @property
    def bytes(self) -> torch.Tensor:
        """Pre-expanded 16 KB UMMA byte blocks."""
        if self._bytes is None:
            self._bytes = torch.empty((max(self.nblocks, 1), 16384), dtype=torch.uint8, device=self.packed.device)
            self.refresh()
        return self._bytes

    def operand(self) -> tuple:
        """(device pointer, a_bits) of the left operand the tiled GEMM reads: the packed
        2 KB blocks (expanded in shared memory by the GEMM, QG_A_BITS=1) or the
        pre-expanded 16 KB byte blocks."""
        if A_BITS:
            return (self.packed.data_ptr(), 1)
        return (self.bytes.data_ptr(), 0)

    def refresh(self):
        """Re-gather + re-expand the blocks (and degrees) from the adjacency's current
        words with the same schedule -- device only, capturable in a CUDA graph."""
        a = self._src
        self.degrees.zero_()
        if self.nblocks:
            if not getattr(self, "_gather", True):      # shipped blocks: expand only
                N.check(_lib().qg_block_prepare(None, self.m, 0, 0, N.ptr(self.blk_rb), N.ptr(self.blk_kt),
                                                self.nblocks, N.ptr(self.packed), N.ptr(self._bytes),
                                                N.ptr(self.degrees), N.stream()), "qg_block_prepare")
                return
            N.check(_lib().qg_block_prepare(N.ptr(a.dwords), a.logical_rows, a.padded_rows, a.padded_cols,
                                            N.ptr(self.blk_rb), N.ptr(self.blk_kt), self.nblocks, N.ptr(self.packed),
                                            N.ptr(self._bytes), N.ptr(self.degrees), N.stream()), "qg_block_prepare")


def blocked(a) -> BlockedAdjacency:
    """Cached BlockedAdjacency of a PackedBitMatrix (built on first use)."""
    if getattr(a, "_blocked", None) is None:
        from .bitgemm import _schedule
        a._blocked = BlockedAdjacency(a, _schedule(a))
    return a._blocked


# ------------------------------------------------------------- code caches
class TiledCodeStack(BitPlaneStack):
    """A plane stack whose source of truth is a tiled u8 code cache.

    ``side`` = "left" (M x K operand, pitch = pad128(rows)) or "right" (K x N
    operand of the NEXT GEMM: rows are K, pitch = npad(cols)).  Plane words are
    built lazily (untile -> bit_qnt) for API consumers and the exact paths.
    """

    def __init__(self, orientation, rows, cols, bits, tiles: torch.Tensor, side: str, pitch: int, pad_to=8):
        pr, pc = padded_dims(rows, cols, orientation, pad_to)
        self.bits = int(bits)
        self._planes = None
        self._meta = (orientation, int(rows), int(cols), int(pr), int(pc))
        self.tiles, self.side, self.pitch = tiles, side, int(pitch)
        self._dwords = None

    def plain_codes(self) -> torch.Tensor:
        rows, cols = self.logical_rows, self.logical_cols
        out = torch.empty((rows, max(cols, 1)), dtype=torch.uint8, device=self.tiles.device)
        if rows * cols:
            N.check(_lib().qg_tiles_to_codes(N.ptr(self.tiles), rows, cols, int(self.side == "right"), self.pitch,
                                             N.ptr(out), out.shape[1], N.stream()), "qg_tiles_to_codes")
        return out

    @property
    def dwords(self) -> torch.Tensor:
        if self._dwords is None:
            o, rows, cols, pr, pc = self._meta
            codes = self.plain_codes()
            words = torch.empty((self.bits, pr * pc // 32), dtype=torch.int32, device=self.tiles.device)
            if words.numel():
                status = N.new_status()
                N.call("qg_quantize_pack", N.ptr(codes), N.SRC_U8, rows, cols, codes.shape[1], 0.0, 1.0, self.bits,
                       N.COLUMN_WISE_ID if o == COLUMN_WISE else N.ROW_WISE_ID, 8, N.ptr(words), None, None, None,
                       N.ptr(status), N.stream())
            self._dwords = words
        return self._dwords

    @dwords.setter
    def dwords(self, value):
        self._dwords = value


def tiles_from_codes(codes: torch.Tensor, rows: int, cols: int, ld: int, side: str) -> tuple:
    """Plain row-major codes [rows][ld] -> (tiled buffer, pitch)."""
    if side == "left":
        pitch = pad128(rows)
        size = pad128(cols) * pitch
    else:
        pitch = npad_of(cols)
        size = pad128(rows) * pitch
    tiles = N.alloc(max(size, 16), torch.uint8, "static")
    if rows * cols:
        N.check(_lib().qg_codes_to_tiles(N.ptr(codes), rows, cols, ld, int(side == "right"), pitch, N.ptr(tiles),
                                         N.stream()), "qg_codes_to_tiles")
    return tiles, pitch


def operand_tiles(stack: BitPlaneStack, side: str, row_sums=None):
    """(tiles, pitch) of an activation stack for use as a left/right operand."""
    if isinstance(stack, TiledCodeStack) and stack.side == side:
        return stack.tiles, stack.pitch
    from .bitpack import stack_code_operand
    rows, cols = stack.logical_rows, stack.logical_cols
    if stack.orientation == ROW_WISE:
        codes, ld = stack_code_operand(stack, colmajor=False, row_sums=row_sums)
    else:
        codes, ld = stack_code_operand(stack, colmajor=False)
    return tiles_from_codes(codes, rows, cols, ld, side)


def weight_tiles(layer, prep):
    """Right-tiled W codes (K = in_dim, N = out_dim), cached on the prepared layer."""
    if getattr(prep, "w_tiles", None) is None:
        dev = prep.w_stack.dwords.device
        wq = torch.empty((layer.in_dim, layer.out_dim), dtype=torch.uint8, device=dev)
        w64 = torch.as_tensor(layer.weight, dtype=torch.float64).to(dev).contiguous()
        tmp = torch.empty_like(prep.w_stack.dwords)
        status = torch.full((1,), N.STATUS_CLEAR, dtype=torch.int64, device=dev)   # one-time, not per forward
        p = layer.weight_params
        N.call("qg_quantize_pack", N.ptr(w64), N.SRC_F64, layer.in_dim, layer.out_dim, layer.out_dim,
               float(p.alpha_min), float(p.scale), p.bits, N.ROW_WISE_ID, 8, N.ptr(tmp), N.ptr(wq), None, None,
               N.ptr(status), N.stream())
        pitch = npad_of(layer.out_dim)
        tiles = torch.zeros(pad128(layer.in_dim) * pitch, dtype=torch.uint8, device=dev)
        N.check(_lib().qg_codes_to_tiles(N.ptr(wq), layer.in_dim, layer.out_dim, layer.out_dim, 1, pitch, N.ptr(tiles),
                                         N.stream()), "qg_codes_to_tiles")
        prep.w_tiles, prep.w_pitch = tiles, pitch
    return prep.w_tiles, prep.w_pitch


# ------------------------------------------------------------ grouped launch
class SegTable:
    """Pinned host segment table + its device copy (captured as one H2D memcpy)."""

    def __init__(self, segs, kind=TSeg):
        n = len(segs)
        self.host = N.alloc(n * ctypes.sizeof(kind), torch.uint8, "host")
        arr = (kind * n).from_address(self.host.data_ptr())
        for i, s in enumerate(segs):
            arr[i] = s
        self.segs = list(segs)
        self.dev = N.alloc(self.host.numel(), torch.uint8, "empty")
        if torch.cuda.is_current_stream_capturing():
            # a captured epoch reuses the same slab addresses every replay, so the table
            # is constant: copy it once after capture (N.flush_static_copies) instead of
            # adding an H2D memcpy node (a PCIe round trip) to every replay
            N.STATIC_COPIES.append((self.dev, self.host))
        else:
            self.dev.copy_(self.host, non_blocking=True)
        self.n = n


def sm_count() -> int:
    return torch.cuda.get_device_properties(N.device()).multi_processor_count


BN_MAX = int(os.environ.get("QG_BN_MAX", "256"))      # tuning experiments


BN_MIN = int(os.environ.get("QG_BN_MIN", "32"))       # tuning experiments


def choose_bn(npad: int, row_blocks_total: int) -> int:
    bn = min(BN_MAX, npad)
    while bn > max(16, BN_MIN) and row_blocks_total * (npad // bn) < 148:
        bn //= 2
    return bn


def use_pair(b_npad: int, row_blocks_total: int, sizes, mode: int) -> bool:
    """2-SM CTA pairs (cta_group::2) for large int32-output stages (the C5 bit-GEMM): each
    CTA stages half of the B tile (needs the operand buffer sizes for the TMA
    descriptors).  The fused-epilogue engine stages stay on single-CTA tiles: measured
    slower in pairs (C4 8.3 vs 7.4 ms/epoch, C3 0.34 vs 0.29 ms; the pair's tile is
    epilogue-bound and 2 CTAs/SM already overlap epilogue with main loop)."""
    return (PAIR and mode == N.GEMM_I32 and sizes is not None and b_npad >= 64
            and row_blocks_total * max(1, b_npad // 256) >= 2 * sm_count())


PAIR_CHAIN = os.environ.get("QG_PAIR_CHAIN", "0") != "0"

# QG_A_BITS=1: adjacency blocks reach the tiled GEMM packed (2 KB per non-zero 128x128
# block instead of 16 KB of 0/1 bytes) and the otherwise idle epilogue warps expand them
# into the ring slot during the main loop: 8x less adjacency traffic from HBM / L2.
A_BITS = os.environ.get("QG_A_BITS", "0") == "1"

# A in tensor memory (default; QG_A_TMEM=0 disables) for large non-chained adjacency
# stages with N tiles <= 128 columns, where TMEM has room beside the accumulator: the
# packed 2 KB blocks are expanded by four warps straight into TENSOR MEMORY (tcgen05.st)
# and the MMAs read A from there (tcgen05.mma [d], [a], b): 8x less adjacency traffic and
# no shared-memory traffic for A.
A_TMEM = os.environ.get("QG_A_TMEM", "1") != "0"


def use_pair_chain(b_npad: int, w_npad: int, row_blocks_total: int, sizes) -> bool:
    """Chained aggregate -> update stages on 2-SM CTA pairs (tc_pair_kernel<.., CHAIN>):
    each CTA streams half of every B / weight tile, so a K tile costs 16 KB + bn*64 B of
    L2 traffic per CTA instead of 16 KB + bn*128 B.  Needs >= 2 pairs per SM of work."""
    return (PAIR_CHAIN and sizes is not None and b_npad >= 64 and w_npad >= 32
            and row_blocks_total >= 2 * sm_count())


def launch(segs, *, a_blocks: bool, b_npad: int, n: int, mode: int, out_layout: int, out_npad: int, epi_struct,
           keep: list, work: float = 0.0, a_bits: bool = False, sizes=None, chain: Chain | None = None):
    """One grouped tiled GEMM over ``segs`` (TSeg list with row_blocks set in .m).
    ``sizes``: per segment (A source bytes, B source bytes), enabling the 2-SM pair path.
    ``chain``: fuse a dense stage-2 GEMM behind this stage (one N tile, see qg_chain)."""
    rbs = [-(-s.m // TILE) for s in segs]
    pair = chain is None and use_pair(b_npad, sum(rbs), sizes, mode) and not a_bits
    if chain is not None:
        if b_npad > 256:
            raise ValueError("chained stage needs one N tile <= 256")
        bn = b_npad
        pair = use_pair_chain(b_npad, chain.w_npad, sum(rbs), sizes) and not a_bits
    elif pair:
        bn = max(64, min(256, b_npad))
    else:
        bn = choose_bn(b_npad, sum(rbs))
    n_tiles = b_npad // bn
    begin = 0
    for s, r in zip(segs, rbs):
        s.cta_begin = begin
        begin += (-(-r // 2) if pair else r) * n_tiles
    if pair:
        begin *= 2                                   # CTAs = 2 x pairs; cta_begin counts pairs
        bh = bn // 2
        for sg, (abytes, bbytes) in zip(segs, sizes):
            N.check(_lib().qg_encode_linear_map(sg.a, abytes, 128, ctypes.byref(sg.tmap_a)), "qg_encode_linear_map")
            N.check(_lib().qg_encode_linear_map(sg.b, bbytes, bh, ctypes.byref(sg.tmap_b)), "qg_encode_linear_map")
    table = SegTable(segs)
    keep.append(table)
    args = TiledArgs()
    args.segs, args.nsegs, args.a_blocks, args.total_ctas = table.dev.data_ptr(), table.n, int(a_blocks), begin
    args.b_npad, args.n, args.bn, args.n_tiles = b_npad, n, bn, n_tiles
    args.mode, args.out_layout, args.out_npad = mode, out_layout, out_npad
    args.a_bits = int(a_bits) if a_blocks else 0
    args.pair = int(pair)
    if epi_struct is not None:
        args.epi = ctypes.pointer(epi_struct)
    if chain is not None:
        args.chain = ctypes.addressof(chain)
        keep.append(chain)
    if not begin:
        return
    global PENDING_JOIN
    if a_blocks and PENDING_JOIN is not None:
        torch.cuda.current_stream().wait_event(PENDING_JOIN)
        PENDING_JOIN = None
    global LAUNCHES
    LAUNCHES += 1
    from . import bitgemm
    if bitgemm.PHASE_HOOK is not None:
        # no memset: a memset node inside a captured epoch would cut the PDL edge between the
        # GEMM launches (every CTA writes all 8 slots; slot 7 is 0 unless the launch is chained)
        stamps = torch.empty((begin, 8), dtype=torch.int64, device=N.device())
        args.phase_ns = stamps.data_ptr()
        bitgemm.PHASE_HOOK.append((stamps, work))
    if bitgemm.PROFILE_HOOK is not None:
        s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_ev.record()
        N.check(_lib().qg_tiled_gemm(args, N.stream()), "qg_tiled_gemm")
        e_ev.record()
        bitgemm.PROFILE_HOOK.append((s_ev, e_ev, work))
        return
    N.check(_lib().qg_tiled_gemm(args, N.stream()), "qg_tiled_gemm")


# ------------------------------------------------------ reduced 1-bit x s-bit
def bmm_reduced(a, x, *, out: torch.Tensor | None = None) -> torch.Tensor:
    """int32 ``reduce_bitplanes(bmm_1bit_by_nbit(a, x))`` in ONE tiled launch.

    The reference computes A.X_p per plane (bitgemm.py:306-371) and then shift-adds
    the planes in int64 (bitgemm.py:282-298).  Since sum_p 2^p X_p is X's code
    matrix, the same int32 result is A . codes(X): the non-zero 128x128 blocks of
    A (zero-tile jumping, bitgemm.py:214-233) times X's right-tiled u8 codes,
    accumulated in TMEM s32.  Exact: the largest entry is (2^s-1)*K < 2^31 for
    K < 8.4M, so _narrow_int32 can never raise here.  Device result, no sync.
    """
    from .bitpack import COLUMN_WISE as _COL, ROW_WISE as _ROW
    from .errors import ShapeError
    if a.orientation != _COL:
        raise ShapeError("left operand must be column-wise packed")
    if x.orientation != _ROW:
        raise ShapeError("right operand must be row-wise packed")
    if a.padded_cols != x.padded_rows or a.logical_cols != x.logical_rows:
        raise ShapeError(f"shared dims mismatch: {a.logical_rows}x{a.logical_cols} vs "
                         f"{x.logical_rows}x{x.logical_cols}")
    m, n = a.logical_rows, x.logical_cols
    if out is None:
        out = N.alloc((m, n), torch.int32, "empty")   # every element is written
    if not (m and n):
        return out
    blk = blocked(a)
    if blk.nblocks == 0:
        out.zero_()
        return out
    xt, _ = operand_tiles(x, "right")
    seg = TSeg()
    a_ptr, a_bits = blk.operand()
    seg.a, seg.b, seg.m, seg.r128 = a_ptr, xt.data_ptr(), m, blk.r128
    seg.blk_count, seg.blk_base, seg.blk_kt = (blk.blk_count.data_ptr(), blk.blk_base.data_ptr(),
                                               blk.blk_kt.data_ptr())
    seg.out_i32 = out.data_ptr()
    keep = []
    # row blocks with no non-zero K tile are written as zeros by the kernel (nk = 0)
    sizes = None if a_bits else [(blk.nblocks * 16384, xt.numel())]
    launch([seg], a_blocks=True, b_npad=npad_of(n), n=n, mode=N.GEMM_I32, out_layout=0, out_npad=0,
           epi_struct=None, keep=keep, work=2.0 * 1024 * (-(-n // 8) * 8) * blk.nz8, a_bits=a_bits, sizes=sizes)
    out._qg_keep = keep           # the segment table must outlive the (async) launch
    return out


# ------------------------------------------------------- grouped entry codes
class EntrySeg(ctypes.Structure):
    """Mirror of ``qg_entry_seg``."""

    _fields_ = [("words", ctypes.c_void_p), ("tiles", ctypes.c_void_p), ("row_sums", ctypes.c_void_p),
                ("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("pr", ctypes.c_int64), ("pc", ctypes.c_int64),
                ("pitch", ctypes.c_int64), ("unit_begin", ctypes.c_int64)]


def entry_tiles(stacks, side: str, want_row_sums: bool, keep: list):
    """Row-wise feature plane stacks of all batches -> tiled codes, ONE launch
    (engine.py:164-176 entry state + orientation fix-up; sum_p 2^p plane_p).
    Returns [(tiles, pitch, row_sums | None)] or None when a stack is not a plain
    row-wise plane stack of a common bit width (callers then convert per batch)."""
    if not stacks or any(type(s) is not BitPlaneStack or s.orientation != ROW_WISE or s.bits != stacks[0].bits
                         for s in stacks):
        return None
    right = side == "right"
    segs, outs, begin = [], [], 0
    # work unit rows: 256 (8 plane words, one 32-byte sector per plane and column) when
    # that still gives >= 2 units per SM, else 32 (small inputs want more CTAs)
    big = sum((-(-s.dims()[2] // 256)) * (-(-(npad_of(s.dims()[1]) if right else s.dims()[3]) // 128))
              for s in stacks) >= 2 * sm_count()
    urows = 256 if big else 32
    for s in stacks:
        rows, cols, pr, pc = s.dims()
        if right:
            pitch = npad_of(cols)
            tiles = N.alloc(max(pad128(rows) * pitch, 16), torch.uint8, "static")
            units = (-(-pr // urows)) * (-(-pitch // 128))
        else:
            pitch = pad128(rows)
            tiles = N.alloc(max(pad128(cols) * pitch, 16), torch.uint8, "static")
            units = (-(-pr // urows)) * (-(-pc // 128))
        rs = N.alloc(rows, torch.int64, "volatile") if (want_row_sums and not right) else None
        seg = EntrySeg()
        seg.words, seg.tiles, seg.row_sums = s.dwords.data_ptr(), tiles.data_ptr(), (rs.data_ptr() if rs is not None
                                                                                     else None)
        seg.rows, seg.cols, seg.pr, seg.pc, seg.pitch, seg.unit_begin = rows, cols, pr, pc, pitch, begin
        begin += units if rows * cols else 0
        segs.append(seg)
        outs.append((tiles, pitch, rs))
        keep.extend([tiles, rs])
    if begin:
        table = SegTable(segs, EntrySeg)
        keep.append(table)
        N.check(N.lib().qg_entry_tiles(table.dev.data_ptr(), len(segs), stacks[0].bits, int(right), urows // 32,
                                       begin, N.stream()), "qg_entry_tiles")
    return outs


# ------------------------------------------------- grouped block expansion
class BlockSeg(ctypes.Structure):
    """Mirror of ``qg_block_seg``."""

    _fields_ = [("packed", ctypes.c_void_p), ("blk_rb", ctypes.c_void_p), ("bytes", ctypes.c_void_p),
                ("degrees", ctypes.c_void_p), ("rows", ctypes.c_int64), ("block_begin", ctypes.c_int64)]


class GroupedRefresh:
    """Per-step block expansion + degrees of many shipped-block batches (QGT3 views) in
    ONE memset + ONE launch, instead of a memset and a launch per batch.  The batches'
    degrees are re-pointed to views of one joint buffer so a single memset zeroes them."""

    def __init__(self, blks: list):
        self.blks = [b for b in blks if b.nblocks]
        dev = N.device()
        total_rows = sum(b.m for b in blks)
        self.degrees = torch.zeros(max(total_rows, 1), dtype=torch.int64, device=dev)
        off = 0
        for b in blks:                              # every batch's degrees -> a view of the joint buffer
            b.degrees = self.degrees[off:off + b.m]
            off += b.m
        segs, begin = [], 0
        for b in self.blks:
            seg = BlockSeg()
            seg.packed, seg.blk_rb = b.packed.data_ptr(), b.blk_rb.data_ptr()
            seg.bytes = b.bytes.data_ptr()
            seg.degrees, seg.rows, seg.block_begin = b.degrees.data_ptr(), b.m, begin
            begin += b.nblocks
            segs.append(seg)
        self.total = begin
        self.keep = []
        if segs:
            n = len(segs)
            host = torch.zeros(n * ctypes.sizeof(BlockSeg), dtype=torch.uint8).pin_memory()
            arr = (BlockSeg * n).from_address(host.data_ptr())
            for i, sg in enumerate(segs):
                arr[i] = sg
            self.table = host.to(dev)                 # static for the runner's lifetime
            self.keep.append(host)
        self.nsegs = len(segs)

    def run(self):
        self.degrees.zero_()
        if self.nsegs:
            N.check(N.lib().qg_block_prepare_grouped(self.table.data_ptr(), self.nsegs, self.total, N.stream()),
                    "qg_block_prepare_grouped")
