"""Any-bitwidth bit-GEMM on B200 (mirror of bitgemm.py).

Compute runs in ``qg_bitgemm`` (csrc/qgtc_gemm.cu): tcgen05.mma kind::i8
over plane stacks recomposed into u8 codes in shared memory, zero-tile
jumping from a per-128-row-block schedule, fused fp64 epilogue.  The Python
layer keeps the reference's signatures, validation order and exceptions.

Scheduling knobs map onto real kernel variants (outputs are invariant, as in
the reference, bitgemm.py:10-16):

* ``jump=True`` runs the zero-tile-jumping schedule built by ``qg_tile_scan``
  (non-zero 128x128-bit blocks only); ``jump=False`` runs every K tile.
* ``reuse=CROSS_TILE`` expands each left tile once for all right planes
  (planes stacked along N, or recomposed into codes); ``CROSS_BIT`` re-expands
  it per plane (one plane per CTA).

These variants apply to ``bmm_1bit_by_nbit`` (and the engine's aggregation
stages).  ``gemm_sbit_by_tbit`` runs one kernel for every knob setting: its
dense s-bit left operand has no zero-tile schedule worth running and its
planes are recomposed into codes once, so ``jump`` / ``reuse`` select only the
reference op counters it reports.

Op counters are the reference's closed forms (bitgemm.py:335-370, 409-461)
over the 8x128 tile flags, computed lazily on the device when read.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _native as N
from .bitpack import (COLUMN_WISE, ROW_WISE, BitPlaneStack, CodeBackedStack, PackedBitMatrix, orient_id, pad128,
                      padded_dims)
from .errors import ReductionOverflowError, ShapeError
from .quantize import QuantParams

CROSS_BIT = "cross-bit"
CROSS_TILE = "cross-tile"

TILE_ROWS = 8
TILE_COLS = 8
TILE_K_BITS = 128
TILE_K_WORDS = TILE_K_BITS // 32

_INT32_MAX = 2 ** 31 - 1
_INT32_MIN = -(2 ** 31)


def popcount32(v) -> np.ndarray:
    """Per-element set-bit count of a uint32 array (bitgemm.py:58-60), on the GPU."""
    arr = np.array(v, dtype=np.uint32, copy=True)
    t = N.to_device(arr.ravel())
    out = torch.empty_like(t)
    N.call("qg_popcount32", N.ptr(t), t.numel(), N.ptr(out), N.stream())
    return out.cpu().numpy().astype(np.uint32).reshape(arr.shape)


@dataclass(eq=False)
class TileMap:
    """Zero/non-zero flags per (row-tile, col-tile); True marks an all-zero tile."""

    row_tiles: int
    col_tiles: int
    flags: np.ndarray


@dataclass
class OpCounters:
    """Exact per-invocation work counts (bitgemm.py:72-89)."""

    tile_mma_count: int = 0
    tile_fetch_count: int = 0
    tiles_skipped: int = 0
    word_and_popcount_count: int = 0
    tiles_total: int = 0

    def __add__(self, other: "OpCounters") -> "OpCounters":
        return OpCounters(
            self.tile_mma_count + other.tile_mma_count,
            self.tile_fetch_count + other.tile_fetch_count,
            self.tiles_skipped + other.tiles_skipped,
            self.word_and_popcount_count + other.word_and_popcount_count,
            self.tiles_total + other.tiles_total,
        )


_tls = threading.local()


def _set_counters(thunk) -> None:
    """Record the last call's counters; ``thunk`` resolves them on demand."""
    _tls.last = thunk


def op_counters() -> OpCounters:
    """Counters of the most recent kernel invocation on this thread (bitgemm.py:95-100)."""
    last = getattr(_tls, "last", None)
    if last is None:
        raise RuntimeError("no bit-GEMM kernel has run on this thread yet")
    if callable(last):
        last = last()
        _tls.last = last
    return replace(last)


@dataclass
class BatchNormParams:
    """Per-output-column batch-norm (bitgemm.py:103-122)."""

    mean: np.ndarray
    var: np.ndarray
    gamma: np.ndarray
    beta: np.ndarray
    eps: float = 1e-5

    def __post_init__(self):
        self.mean = np.asarray(self.mean, dtype=np.float64)
        self.var = np.asarray(self.var, dtype=np.float64)
        self.gamma = np.asarray(self.gamma, dtype=np.float64)
        self.beta = np.asarray(self.beta, dtype=np.float64)
        n = len(self.mean)
        if any(len(a) != n for a in (self.var, self.gamma, self.beta)):
            raise ValueError("batch-norm parameter vectors disagree on length")
        if not (self.var + self.eps > 0).all():
            raise ValueError("Var + eps must be positive for every column")

    def denom(self) -> np.ndarray:
        # np.sqrt is correctly rounded, like the reference's expression (bitgemm.py:201)
        return np.sqrt(self.var + self.eps)


@dataclass
class EpilogueSpec:
    """Fused post-processing of an integer accumulator (bitgemm.py:125-153)."""

    kind: str = "none"
    lhs_params: QuantParams | None = None
    rhs_params: QuantParams | None = None
    lhs_row_sums: object = None
    rhs_col_sums: object = None
    inner_dim: int = 0
    bias: np.ndarray | None = None
    bn: BatchNormParams | None = None
    out_params: QuantParams | None = None

    def __post_init__(self):
        if self.kind not in ("none", "relu", "tanh", "batch-norm"):
            raise ValueError(f"unknown epilogue kind {self.kind!r}")
        if self.kind == "batch-norm" and self.bn is None:
            raise ValueError("kind='batch-norm' requires bn parameters")


# ------------------------------------------------------- epilogue plumbing
class _EpiPlan:
    """ctypes epilogue struct + the device tensors it points at + outputs."""

    def __init__(self):
        self.keep = []
        self.struct = N.Epilogue()
        self.out_real = None
        self.out_stack = None
        self.row_sums = None
        self.status = None


def _dev_vec(x, dtype, n=None):
    if x is None:
        return None
    t = N.to_device(x if isinstance(x, torch.Tensor) else np.asarray(x), dtype)
    return t


def _build_epilogue(epi: EpilogueSpec, rows: int, cols: int, *, out_orientation=ROW_WISE,
                    out_pad_to=8, want_row_sums=False, dev=None) -> _EpiPlan:
    """Validate like apply_epilogue (bitgemm.py:156-211) and prepare device state."""
    amb = epi.rhs_params.alpha_min if epi.rhs_params is not None else 0.0
    ama = epi.lhs_params.alpha_min if epi.lhs_params is not None else 0.0
    if amb != 0.0 and epi.lhs_row_sums is None:
        raise ValueError("rhs alpha_min != 0 requires lhs_row_sums")
    if ama != 0.0 and epi.rhs_col_sums is None:
        raise ValueError("lhs alpha_min != 0 requires rhs_col_sums")
    bias = None
    if epi.bias is not None:
        bias = epi.bias if isinstance(epi.bias, torch.Tensor) else np.asarray(epi.bias, dtype=np.float64)
        if tuple(bias.shape) != (cols,):
            raise ValueError("bias length must match output columns")
    bn = None
    if epi.bn is not None:
        if len(epi.bn.mean) != cols:
            raise ValueError("batch-norm column count must match output columns")
        bn = (epi.bn.mean, epi.bn.denom(), epi.bn.gamma, epi.bn.beta)
    kind = epi.kind if epi.kind in ("relu", "tanh") else "none"
    return _build_epilogue_raw(epi.lhs_params, epi.rhs_params, epi.lhs_row_sums, epi.rhs_col_sums,
                               epi.inner_dim, bias, bn, kind, epi.out_params, rows, cols, out_orientation,
                               out_pad_to, want_row_sums, dev or N.device())


def _build_epilogue_raw(lhs_params, rhs_params, row_sums, col_sums, inner_dim, bias, bn, kind, out_params,
                        rows, cols, out_orientation, out_pad_to, want_row_sums, dev, code_cache=False) -> _EpiPlan:
    """Device epilogue state; fp64 coefficients grouped as _dequantize (bitgemm.py:166-178)."""
    plan = _EpiPlan()
    e = plan.struct
    ama, sa = (0.0, 1.0) if lhs_params is None else (lhs_params.alpha_min, lhs_params.scale)
    amb, sb = (0.0, 1.0) if rhs_params is None else (rhs_params.alpha_min, rhs_params.scale)
    e.k_acc = sa * sb
    if amb != 0.0:
        rs = _dev_vec(row_sums, torch.int64)
        plan.keep.append(rs)
        e.use_row, e.k_row = 1, sa * amb
        e.row_sums = rs.data_ptr() if rs is not None else None     # None: set per segment
    if ama != 0.0:
        cs = _dev_vec(col_sums, torch.int64)
        plan.keep.append(cs)
        e.use_col, e.k_col = 1, sb * ama
        e.col_sums = cs.data_ptr() if cs is not None else None
    if ama != 0.0 and amb != 0.0:
        e.use_const, e.k_const = 1, (float(inner_dim) * ama) * amb
    if bias is not None:
        b = _dev_vec(bias, torch.float64)
        plan.keep.append(b)
        e.bias = b.data_ptr()
    if bn is not None:
        vecs = [_dev_vec(v, torch.float64) for v in bn]
        if len(vecs) == 4:   # RN(1/denom): IEEE division on the host side of the contract
            vecs.append(1.0 / vecs[1])
        plan.keep.extend(vecs)
        e.bn_mean, e.bn_denom, e.bn_gamma, e.bn_beta, e.bn_inv_denom = (v.data_ptr() for v in vecs)
    e.act = N.ACT[kind]
    if out_params is None:
        plan.out_real = N.alloc((rows, cols), torch.float64, "empty")
        e.out_kind, e.out_real = N.OUT_REAL, plan.out_real.data_ptr()
        return plan
    q = out_params
    pr, pc = padded_dims(rows, cols, out_orientation, out_pad_to)
    e.out_kind, e.q_bits, e.q_amin, e.q_scale = N.OUT_PLANES, q.bits, q.alpha_min, q.scale
    e.q_inv_scale = 1.0 / q.scale
    e.q_orientation, e.q_prows, e.q_pcols = orient_id(out_orientation), pr, pc
    if code_cache:
        # codes only, in the next GEMM's operand layout: a column-wise output feeds a left
        # operand (row-major codes), a row-wise output a right operand (col-major codes)
        colmajor = out_orientation == ROW_WISE
        ld = pad128(rows if colmajor else cols)
        codes = N.alloc(((cols if colmajor else rows), ld), torch.uint8, "static")
        plan.out_stack = CodeBackedStack(out_orientation, rows, cols, q.bits, codes, ld, colmajor, out_pad_to)
        e.q_codes, e.q_codes_ld, e.q_codes_colmajor, e.q_skip_planes = codes.data_ptr(), ld, int(colmajor), 1
        e.q_planes = 0
    else:
        planes = N.alloc((q.bits, pr * pc // 32), torch.int32, "volatile")
        plan.out_stack = BitPlaneStack._wrap(out_orientation, rows, cols, pr, pc, planes)
        e.q_planes = planes.data_ptr()
    if want_row_sums:
        plan.row_sums = N.alloc(rows, torch.int64, "volatile")
        e.q_row_sums = plan.row_sums.data_ptr()
    plan.status = N.new_status()
    e.status = plan.status.data_ptr()
    return plan


def _finish_epilogue(plan: _EpiPlan, cols: int, check: bool = True):
    if plan.out_stack is None:
        return plan.out_real
    if check:
        N.raise_nonfinite(plan.status, cols)
    return plan.out_stack


def apply_epilogue(acc, epi: EpilogueSpec, *, out_orientation: str = ROW_WISE, out_pad_to: int = 8):
    """Dequantize, bias, batch-norm, activate, optionally requantize (bitgemm.py:182-211).

    Returns a float64 numpy matrix, or a device-resident BitPlaneStack when
    ``epi.out_params`` is set.  The fused GEMM path evaluates the same device
    function, so fused and standalone epilogues agree bit for bit.
    """
    if isinstance(acc, torch.Tensor):
        t = acc.to(N.device())
    else:
        t = N.to_device(np.asarray(acc))
    if t.dim() != 2:
        raise ValueError("accumulator must be 2-D")
    rows, cols = t.shape
    if t.dtype != torch.int32 and t.numel():
        # the kernel reads int32 accumulators: refuse values that would not survive the
        # narrowing (the reference dequantizes acc.astype(float64), bitgemm.py:156-160)
        lo, hi = torch.iinfo(torch.int32).min, torch.iinfo(torch.int32).max
        if t.is_floating_point():
            bad = ~torch.isfinite(t) | (t != torch.trunc(t)) | (t < lo) | (t > hi)
        else:
            bad = (t < lo) | (t > hi)
        if bool(bad.any()):
            raise ReductionOverflowError("accumulator values must be integers that fit int32 "
                                         "(the device epilogue reads int32 accumulators)")
    plan = _build_epilogue(epi, rows, cols, out_orientation=out_orientation, out_pad_to=out_pad_to,
                           dev=t.device)
    t32 = t.to(torch.int32).contiguous()
    N.check(N.lib().qg_epilogue_apply(N.ptr(t32), rows, cols, plan.struct, N.stream()), "apply_epilogue")
    out = _finish_epilogue(plan, cols)
    return out.cpu().numpy() if isinstance(out, torch.Tensor) else out


# ------------------------------------------------------------- tile scans
class _Schedule:
    """Zero-tile-jumping schedule + scan products of one column-wise 1-bit operand."""

    def __init__(self, a: PackedBitMatrix):
        dev = a.dwords.device
        pr, pc = a.padded_rows, a.padded_cols
        self.rt, self.ct = pr // TILE_ROWS, pc // TILE_K_BITS
        nrb = -(-pr // 128)
        self.flags = N.alloc((self.rt, self.ct), torch.uint8, "empty")
        self.degrees = N.alloc(a.logical_rows, torch.int64, "volatile")
        self.zero_count = N.alloc(1, torch.int64, "volatile")
        self.blk_list = N.alloc((nrb, max(self.ct, 1)), torch.int32, "empty")
        self.blk_count = N.alloc(nrb, torch.int32, "volatile")
        self._zeros = None
        if a.dwords.numel() == 0:
            self.degrees.zero_()
            return
        N.call("qg_tile_scan", N.ptr(a.dwords), a.logical_rows, pr, pc, N.ptr(self.flags), N.ptr(self.degrees),
               N.ptr(self.zero_count), N.ptr(self.blk_list), N.ptr(self.blk_count), N.stream())
        self._zeros = None

    @property
    def zeros(self) -> int:
        if self._zeros is None:
            self._zeros = int(self.zero_count.item())
        return self._zeros


def _schedule(a: PackedBitMatrix) -> _Schedule:
    if a._schedule is None:
        a._schedule = _Schedule(a)
    return a._schedule


def scan_zero_tiles(a: PackedBitMatrix) -> TileMap:
    """Flag all-zero 8x128 tiles of a column-wise 1-bit matrix (bitgemm.py:214-233).  Cached."""
    if a.orientation != COLUMN_WISE:
        raise ShapeError("zero-tile scan expects a column-wise operand")
    if a._tilemap is not None:
        return a._tilemap
    s = _schedule(a)
    rt, ct = s.rt, s.ct
    if rt and ct:
        flags = s.flags.cpu().numpy().astype(bool)
    else:
        flags = np.zeros((rt, ct), dtype=bool)
    tm = TileMap(row_tiles=rt, col_tiles=ct, flags=flags)
    a._tilemap = tm
    return tm


def _plane_zero_tiles(stack: BitPlaneStack) -> list[int]:
    out = torch.zeros(stack.bits, dtype=torch.int64, device=stack.dwords.device)
    N.call("qg_plane_zero_tiles", N.ptr(stack.dwords), stack.bits, stack.padded_rows, stack.padded_cols,
           N.ptr(out), N.stream())
    return [int(v) for v in out.cpu()]


# --------------------------------------------------------------- the GEMM
PROFILE_HOOK = None   # bench.py: list receiving (start_event, end_event, algorithmic_ops) per launch
PHASE_HOOK = None     # tools/: list receiving (grid_ctas, int64 [ctas, 6] %globaltimer stamps) per launch


def _launch_work(mp, kp, np_, rbits, mode, schedule):
    """Algorithmic int8-MAC ops of one launch: 2 x 1024 x N_padded per non-zero 8x128 left tile."""
    tiles = (mp // TILE_ROWS) * (kp // TILE_K_BITS)
    if schedule is not None:
        tiles -= schedule.zeros
    return 2.0 * 1024 * np_ * tiles * (rbits if mode == N.GEMM_PER_PLANE else 1)


def gemm_device(lhs_dwords, lbits, m, mp, k, kp, rhs_dwords, rbits, n, np_, *, mode, schedule=None,
                out=None, epi_struct=None, algo="auto", cross_bit=False, overflow=None, scratch=None,
                lhs_codes=None, rhs_codes=None, entry: str = "qg_bitgemm"):
    """Launch qg_bitgemm on device tensors (no syncs).  ``lhs_codes``/``rhs_codes``
    are optional (u8 tensor, ld) code caches used instead of the plane words."""
    args = N.GemmArgs()
    if lhs_codes is not None:
        args.lhs_codes, args.lhs_ld = lhs_codes[0].data_ptr(), lhs_codes[1]
    if rhs_codes is not None:
        args.rhs_codes, args.rhs_ld = rhs_codes[0].data_ptr(), rhs_codes[1]
    args.lhs, args.lbits, args.m, args.m_padded, args.k, args.k_padded = \
        (lhs_dwords.data_ptr() if lhs_dwords is not None else args.lhs_codes), lbits, m, mp, k, kp
    args.rhs, args.rbits, args.n, args.n_padded = \
        (rhs_dwords.data_ptr() if rhs_dwords is not None else args.rhs_codes), rbits, n, np_
    if schedule is not None:
        args.blk_list, args.blk_count = schedule.blk_list.data_ptr(), schedule.blk_count.data_ptr()
    args.mode, args.algo, args.cross_bit = mode, N.ALGO[algo], int(cross_bit)
    if out is not None:
        args.out_i32 = out.data_ptr()
    if epi_struct is not None:
        args.epi = ctypes_pointer(epi_struct)
    if overflow is not None:
        args.overflow = overflow.data_ptr()
    if scratch is not None:
        args.scratch_i32 = scratch.data_ptr()
    if PHASE_HOOK is not None:
        ctas = max(1, (mp + 127) // 128) * 64
        stamps = torch.zeros((ctas, 70), dtype=torch.int64, device=N.device())
        args.phase_ns = stamps.data_ptr()
        PHASE_HOOK.append(stamps)
    if PROFILE_HOOK is not None:
        s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_ev.record()
        N.check(getattr(N.lib(), entry)(args, N.stream()), entry)
        e_ev.record()
        PROFILE_HOOK.append((s_ev, e_ev, _launch_work(mp, kp, np_, rbits, mode, schedule)))
        return
    N.check(getattr(N.lib(), entry)(args, N.stream()), entry)


def ctypes_pointer(struct):
    import ctypes
    return ctypes.pointer(struct)


def needs_exact_path(lbits: int, rbits: int, k: int) -> bool:
    """True when the s32 tensor accumulator could wrap (qg_bitgemm picks POPC)."""
    return ((1 << lbits) - 1) * ((1 << rbits) - 1) * k >= _INT32_MAX


def _check_reuse(reuse: str):
    if reuse not in (CROSS_BIT, CROSS_TILE):
        raise ValueError(f"reuse must be {CROSS_BIT!r} or {CROSS_TILE!r}")


def _c_counters(fn: str, *args) -> OpCounters:
    """OpCounters from the C-ABI closed forms (qg_bmm_counters / qg_gemm_counters)."""
    import ctypes
    out = (ctypes.c_int64 * 5)()
    N.check(getattr(N.lib(), fn)(*args, ctypes.byref(out)), fn)
    return OpCounters(*(int(v) for v in out))


def _bmm_counters(a: PackedBitMatrix, s: int, n_chunks: int, jump: bool, reuse: str):
    """Counters of bmm_1bit_by_nbit (bitgemm.py:335-370); resolved lazily (needs the scan)."""
    def resolve():
        sch = _schedule(a)
        zeros = sch.zeros if (jump and sch.rt * sch.ct) else 0
        return _c_counters("qg_bmm_counters", sch.rt, sch.ct, zeros, s, n_chunks, int(jump),
                           int(reuse == CROSS_TILE))
    return resolve


def bmm_1bit_by_nbit(a: PackedBitMatrix, x: BitPlaneStack, *, jump: bool = True,
                     reuse: str = CROSS_TILE) -> list[np.ndarray]:
    """1-bit by s-bit product, one int32 matrix per plane of X (bitgemm.py:306-371)."""
    outs = bmm_planes_device(a, x, jump=jump, reuse=reuse)
    host = outs.cpu().numpy()
    return [host[p] for p in range(x.bits)]


def bmm_planes_device(a: PackedBitMatrix, x: BitPlaneStack, *, jump=True, reuse=CROSS_TILE,
                      algo="auto") -> torch.Tensor:
    _check_reuse(reuse)
    if a.orientation != COLUMN_WISE:
        raise ShapeError("left operand must be column-wise packed")
    if x.orientation != ROW_WISE:
        raise ShapeError("right operand must be row-wise packed")
    if a.padded_cols != x.padded_rows or a.logical_cols != x.logical_rows:
        raise ShapeError(f"shared dims mismatch: {a.logical_rows}x{a.logical_cols} vs "
                         f"{x.logical_rows}x{x.logical_cols}")
    s, m, n = x.bits, a.logical_rows, x.logical_cols
    out = torch.zeros((s, m, n), dtype=torch.int32, device=a.dwords.device)
    sch = _schedule(a) if jump else None
    if m and n and a.padded_cols:
        gemm_device(a.dwords, 1, m, a.padded_rows, a.logical_cols, a.padded_cols, x.dwords, s, n,
                    x.padded_cols, mode=N.GEMM_PER_PLANE, schedule=sch, out=out, algo=algo,
                    cross_bit=(reuse == CROSS_BIT), entry="qg_bmm_1xs")
    _set_counters(_bmm_counters(a, s, x.padded_cols // TILE_COLS, jump, reuse))
    return out


def _narrow_int32(total: np.ndarray) -> np.ndarray:
    if total.size and (total.max() > _INT32_MAX or total.min() < _INT32_MIN):
        raise ReductionOverflowError(f"reduced value {int(total.max())} does not fit a signed 32-bit output")
    return total.astype(np.int32)


def reduce_bitplanes(plane_accs) -> np.ndarray:
    """Shifted 64-bit reduction sum_p acc_p << p narrowed to int32 (bitgemm.py:291-298)."""
    if not len(plane_accs):
        raise ValueError("nothing to reduce")
    if isinstance(plane_accs, torch.Tensor):
        t = plane_accs.to(N.device(), torch.int64)
    else:
        t = torch.stack([N.to_device(np.asarray(acc), torch.int64) if not isinstance(acc, torch.Tensor)
                         else acc.to(N.device(), torch.int64) for acc in plane_accs])
    shape = tuple(t.shape[1:])
    flat = t.reshape(t.shape[0], -1).contiguous()
    out = torch.empty(flat.shape[1], dtype=torch.int32, device=flat.device)
    flag = torch.zeros(1, dtype=torch.int32, device=flat.device)
    N.call("qg_reduce_planes", N.ptr(flat), flat.shape[0], flat.shape[1], N.ptr(out), N.ptr(flag), N.stream())

    def peak():
        sh = torch.arange(flat.shape[0], device=flat.device, dtype=torch.int64)
        return int((flat << sh[:, None]).sum(dim=0).max().item())
    N.raise_overflow(flag, peak)
    return out.reshape(shape).cpu().numpy()


def _gemm_counters(x: BitPlaneStack, t: int, n_chunks: int, jump: bool, reuse: str):
    def resolve():
        import ctypes
        rt, ct = x.padded_rows // TILE_ROWS, x.padded_cols // TILE_K_BITS
        zeros = _plane_zero_tiles(x) if (jump and rt * ct) else [0] * x.bits
        return _c_counters("qg_gemm_counters", rt, ct, (ctypes.c_int64 * x.bits)(*zeros), x.bits, t, n_chunks,
                           int(jump), int(reuse == CROSS_TILE))
    return resolve


def _check_gemm_operands(x: BitPlaneStack, w: BitPlaneStack):
    if x.orientation != COLUMN_WISE:
        raise ShapeError("left stack must be column-wise packed")
    if w.orientation != ROW_WISE:
        raise ShapeError("right stack must be row-wise packed")
    if not (1 <= x.bits <= 8 and 1 <= w.bits <= 8):
        raise ValueError("operand bit counts must be in [1, 8]")
    if x.padded_cols != w.padded_rows or x.logical_cols != w.logical_rows:
        raise ShapeError(f"inner dims mismatch: {x.logical_rows}x{x.logical_cols} vs "
                         f"{w.logical_rows}x{w.logical_cols}")


def gemm_sbit_by_tbit(x: BitPlaneStack, w: BitPlaneStack, out: str = "int32",
                      epi: EpilogueSpec | None = None, *, jump: bool = True,
                      reuse: str = CROSS_TILE, out_orientation: str = ROW_WISE,
                      out_pad_to: int = 8, clock=None):
    """s-bit by t-bit product with optional fused epilogue (bitgemm.py:374-475).

    ``out="int32"`` returns the int32 accumulator (numpy); ``out="bitplanes"``
    runs the epilogue inside the GEMM kernel and returns a device-resident
    BitPlaneStack.  Overflow of the int32 result raises, never wraps.
    """
    _check_reuse(reuse)
    if out not in ("int32", "bitplanes"):
        raise ValueError(f"out must be 'int32' or 'bitplanes', got {out!r}")
    _check_gemm_operands(x, w)
    if out == "int32" and epi is not None:
        raise ValueError("out='int32' returns the raw accumulator; "
                         "apply the epilogue separately or use out='bitplanes'")
    if out == "bitplanes" and (epi is None or epi.out_params is None):
        raise ValueError("out='bitplanes' requires an epilogue with out_params")
    m, n, k = x.logical_rows, w.logical_cols, x.logical_cols
    dev = x.dwords.device
    overflow = torch.zeros(1, dtype=torch.int32, device=dev)
    exact = needs_exact_path(x.bits, w.bits, k)
    if out == "int32":
        acc = torch.zeros((m, n), dtype=torch.int32, device=dev)
        if m and n:
            gemm_device(x.dwords, x.bits, m, x.padded_rows, k, x.padded_cols, w.dwords, w.bits, n, w.padded_cols,
                        mode=N.GEMM_I32, out=acc, overflow=overflow, entry="qg_gemm_sxt")
        _set_counters(_gemm_counters(x, w.bits, w.padded_cols // TILE_COLS, jump, reuse))
        if exact:
            N.raise_overflow(overflow, lambda: _peak(x, w))
        return acc.cpu().numpy()
    plan = _build_epilogue(epi, m, n, out_orientation=out_orientation, out_pad_to=out_pad_to, dev=dev)
    scratch = torch.empty((m, n), dtype=torch.int32, device=dev) if exact else None
    if m and n:
        gemm_device(x.dwords, x.bits, m, x.padded_rows, k, x.padded_cols, w.dwords, w.bits, n, w.padded_cols,
                    mode=N.GEMM_EPILOGUE, epi_struct=plan.struct, overflow=overflow, scratch=scratch,
                    entry="qg_gemm_sxt")
    _set_counters(_gemm_counters(x, w.bits, w.padded_cols // TILE_COLS, jump, reuse))
    if exact:
        N.raise_overflow(overflow, lambda: _peak(x, w))
    return _finish_epilogue(plan, n)


def _peak(x: BitPlaneStack, w: BitPlaneStack) -> int:
    from .bitpack import stack_codes
    a = stack_codes(x).to(torch.float64)
    b = stack_codes(w).to(torch.float64)
    return int((a @ b).max().item())


def mma_tile_1bit(a_tile, b_tile, acc) -> np.ndarray:
    """One 8x128x8 tile MMA, acc updated in place (bitgemm.py:236-253)."""
    a = np.asarray(a_tile, dtype=np.uint32)
    b = np.asarray(b_tile, dtype=np.uint32)
    acc = np.asarray(acc)
    if a.shape != (TILE_ROWS, TILE_K_WORDS):
        raise ShapeError(f"a_tile must be (8, 4) words, got {a.shape}")
    if b.shape != (TILE_K_WORDS, TILE_COLS):
        raise ShapeError(f"b_tile must be (4, 8) words, got {b.shape}")
    if acc.shape != (TILE_ROWS, TILE_COLS):
        raise ShapeError(f"acc must be (8, 8), got {acc.shape}")
    lhs = PackedBitMatrix(COLUMN_WISE, 8, 128, 8, 128, a.ravel())
    rhs = BitPlaneStack._wrap(ROW_WISE, 128, 8, 128, 8, N.to_device(np.ascontiguousarray(b.T).ravel()).view(1, -1))
    prod = torch.zeros((1, 8, 8), dtype=torch.int32, device=lhs.dwords.device)
    gemm_device(lhs.dwords, 1, 8, 8, 128, 128, rhs.dwords, 1, 8, 8, mode=N.GEMM_PER_PLANE, out=prod)
    acc += prod[0].cpu().numpy().astype(acc.dtype)
    return acc
