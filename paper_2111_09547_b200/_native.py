"""ctypes binding of the in-tree C-ABI library ``_lib/libqgtc_b200.so``.

The library exports the entry points declared in ``include/qgtc_b200.h``.
There is no CPU fallback: if the library or a CUDA device is missing, every
compute call raises ``RuntimeError`` loudly.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from .errors import DataError, ReductionOverflowError, ShapeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libqgtc_b200.so")

QG_OK, QG_ERR_ARG, QG_ERR_SHAPE, QG_ERR_BITS, QG_ERR_CUDA, QG_ERR_UNSUPPORTED = range(6)
COLUMN_WISE_ID, ROW_WISE_ID = 0, 1
SRC_F32, SRC_F64, SRC_U8 = 0, 1, 2
ACT = {"none": 0, "relu": 1, "tanh": 2}
OUT_REAL, OUT_PLANES = 0, 1
GEMM_PER_PLANE, GEMM_I32, GEMM_EPILOGUE = 0, 1, 2
ALGO = {"auto": 0, "tcgen05": 1, "popc": 2}

STATUS_CLEAR = 0x7F7F7F7F7F7F7F7F

# every compute entry point declared in include/qgtc_b200.h
EXPORTS = ("qg_version", "qg_status_reset", "qg_quantize_pack", "qg_pack_planes", "qg_unpack", "qg_repack",
           "qg_tile_scan", "qg_plane_zero_tiles", "qg_epilogue_apply", "qg_bitgemm", "qg_reduce_planes",
           "qg_popcount32", "qg_edges_to_bits", "qg_test_div", "qg_planes_to_codes",
           "qg_test_requant", "qg_tiled_gemm", "qg_block_prepare", "qg_codes_to_tiles",
           "qg_tiles_to_codes", "qg_entry_tiles",
           "qg_block_prepare_grouped", "qg_bmm_1xs", "qg_gemm_sxt", "qg_batch_h2d", "qg_bmm_counters",
           "qg_gemm_counters", "qg_encode_linear_map", "qg_slab_reset", "qg_partition_bfs")

_vp, _i64, _i32, _f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double


class Epilogue(ctypes.Structure):
    """Mirror of ``qg_epilogue`` (include/qgtc_b200.h)."""

    _fields_ = [
        ("act", ctypes.c_int32), ("use_row", ctypes.c_int32), ("use_col", ctypes.c_int32),
        ("use_const", ctypes.c_int32),
        ("k_acc", _f64), ("k_row", _f64), ("k_col", _f64), ("k_const", _f64),
        ("row_sums", _vp), ("col_sums", _vp), ("bias", _vp),
        ("bn_mean", _vp), ("bn_denom", _vp), ("bn_gamma", _vp), ("bn_beta", _vp), ("bn_inv_denom", _vp),
        ("q_inv_scale", _f64), ("out_kind", ctypes.c_int32), ("q_bits", ctypes.c_int32),
        ("q_amin", _f64), ("q_scale", _f64),
        ("q_orientation", ctypes.c_int32), ("pad_", ctypes.c_int32),
        ("q_prows", _i64), ("q_pcols", _i64),
        ("out_real", _vp), ("q_planes", _vp), ("q_row_sums", _vp), ("status", _vp),
        ("q_codes", _vp), ("q_codes_ld", _i64), ("q_codes_colmajor", ctypes.c_int32),
        ("q_skip_planes", ctypes.c_int32), ("screen_rmax", _f64), ("reserved_d1", _f64),
    ]


class GemmArgs(ctypes.Structure):
    """Mirror of ``qg_gemm_args`` (include/qgtc_b200.h)."""

    _fields_ = [
        ("lhs", _vp), ("lbits", ctypes.c_int32), ("pad0", ctypes.c_int32),
        ("m", _i64), ("m_padded", _i64), ("k", _i64), ("k_padded", _i64),
        ("rhs", _vp), ("rbits", ctypes.c_int32), ("pad1", ctypes.c_int32),
        ("n", _i64), ("n_padded", _i64),
        ("blk_list", _vp), ("blk_count", _vp),
        ("mode", ctypes.c_int32), ("algo", ctypes.c_int32),
        ("out_i32", _vp), ("epi", ctypes.POINTER(Epilogue)), ("overflow", _vp), ("scratch_i32", _vp),
        ("lhs_codes", _vp), ("lhs_ld", _i64), ("rhs_codes", _vp), ("rhs_ld", _i64),
        ("phase_ns", _vp), ("cross_bit", ctypes.c_int32), ("pad2", ctypes.c_int32),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    """Load the native library (once).  Raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"native library missing: {LIB_PATH} (run __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        sigs = {
            "qg_version": ([], ctypes.c_int),
            "qg_status_reset": ([_vp, _i64, _vp], ctypes.c_int),
            "qg_slab_reset": ([_vp, _i64, _vp, _i64, _vp], ctypes.c_int),
            "qg_quantize_pack": ([_vp, _i32, _i64, _i64, _i64, _f64, _f64, _i32, _i32, _i32, _vp, _vp, _vp, _vp,
                                  _vp, _vp], ctypes.c_int),
            "qg_pack_planes": ([_vp, _i64, _i64, _i64, _i32, _i32, _vp, _vp, _vp], ctypes.c_int),
            "qg_unpack": ([_vp, _i64, _i64, _i64, _i64, _i64, _i32, _vp, _vp, _vp], ctypes.c_int),
            "qg_repack": ([_vp, _i64, _i64, _i64, _i32, _vp, _i64, _i64, _vp], ctypes.c_int),
            "qg_tile_scan": ([_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
            "qg_plane_zero_tiles": ([_vp, _i64, _i64, _i64, _vp, _vp], ctypes.c_int),
            "qg_epilogue_apply": ([_vp, _i64, _i64, ctypes.POINTER(Epilogue), _vp], ctypes.c_int),
            "qg_bitgemm": ([ctypes.POINTER(GemmArgs), _vp], ctypes.c_int),
            "qg_bmm_1xs": ([ctypes.POINTER(GemmArgs), _vp], ctypes.c_int),
            "qg_gemm_sxt": ([ctypes.POINTER(GemmArgs), _vp], ctypes.c_int),
            "qg_reduce_planes": ([_vp, _i64, _i64, _vp, _vp, _vp], ctypes.c_int),
            "qg_popcount32": ([_vp, _i64, _vp, _vp], ctypes.c_int),
            "qg_edges_to_bits": ([_vp, _vp, _i64, _i64, _vp, _i64, _i64, _vp], ctypes.c_int),
            "qg_test_div": ([_vp, _vp, _vp, _i64, _vp, _vp, _vp], ctypes.c_int),
            "qg_test_requant": ([_vp, _i64, _f64, _f64, _f64, _i32, _vp, _vp, _vp], ctypes.c_int),
            "qg_planes_to_codes": ([_vp, _i64, _i64, _i64, _i64, _i64, _i32, _vp, _i64, _i32, _vp, _vp],
                                   ctypes.c_int),
            "qg_entry_tiles": ([_vp, _i32, _i32, _i32, _i32, _i64, _vp], ctypes.c_int),
            "qg_block_prepare_grouped": ([_vp, _i32, _i64, _vp], ctypes.c_int),
            "qg_batch_h2d": ([_vp, _i64, _vp, _vp], ctypes.c_int),
            "qg_bmm_counters": ([_i64, _i64, _i64, _i32, _i64, _i32, _i32, _vp], ctypes.c_int),
            "qg_gemm_counters": ([_i64, _i64, _vp, _i32, _i32, _i64, _i32, _i32, _vp], ctypes.c_int),
            "qg_partition_bfs": ([_i64, _vp, _vp, _i64, _i64, _vp], ctypes.c_int),
        }
        for name, (argt, rest) in sigs.items():
            fn = getattr(L, name)
            fn.argtypes = argt
            fn.restype = rest
        _lib = L
    return _lib


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2111_09547_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> ctypes.c_void_p | None:
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def check(rc: int, what: str) -> None:
    if rc == QG_OK:
        return
    if rc == QG_ERR_SHAPE:
        raise ShapeError(f"{what}: incompatible operand shapes")
    if rc == QG_ERR_BITS:
        raise ValueError(f"{what}: bit width outside [1, 8]")
    if rc == QG_ERR_ARG:
        raise ValueError(f"{what}: invalid argument")
    if rc == QG_ERR_UNSUPPORTED:
        raise RuntimeError(f"{what}: shape not supported by the selected algorithm")
    raise RuntimeError(f"{what}: CUDA launch failed ({torch.cuda.get_device_name()})")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


# ------------------------------------------------------------ allocation
# Every per-forward device buffer is requested through ALLOC with a kind:
#   "static"   -- zero-initialised once (code caches: padding must stay zero,
#                  the valid region is fully rewritten by every forward)
#   "volatile" -- must be zero at the start of every forward (atomic accumulators)
#   "empty"    -- fully written by its producer
#   "status"   -- first-bad-index cells, reset to STATUS_CLEAR every forward
# The default allocator is plain torch; runtime.EpochRunner records the sequence
# once and then serves it from persistent slabs, so a captured epoch has ONE
# memset + ONE fill instead of a fill kernel per buffer.
class TorchAlloc:
    def take(self, shape, dtype, kind):
        if kind == "host":
            # pageable staging: torch makes pageable H2D copies synchronous w.r.t. the
            # host buffer, so eager callers may drop it right after the copy
            return torch.empty(shape, dtype=dtype)
        dev = device()
        if kind == "status":
            return torch.full(shape, STATUS_CLEAR, dtype=torch.int64, device=dev)
        if kind == "empty":
            return torch.empty(shape, dtype=dtype, device=dev)
        return torch.zeros(shape, dtype=dtype, device=dev)


ALLOC = TorchAlloc()

# (device, pinned host) pairs whose contents are fixed for the lifetime of a captured
# graph (segment tables); copied once right after capture by flush_static_copies()
STATIC_COPIES: list = []


def flush_static_copies() -> None:
    while STATIC_COPIES:
        dev, host = STATIC_COPIES.pop()
        dev.copy_(host)
    torch.cuda.synchronize()


def alloc(shape, dtype, kind="static") -> torch.Tensor:
    shape = tuple(int(v) for v in (shape if isinstance(shape, (tuple, list)) else (shape,)))
    return ALLOC.take(shape, dtype, kind)


class SlabPlan:
    """Records the allocation sequence of one forward (torch-backed)."""

    def __init__(self):
        self.seq = []

    def take(self, shape, dtype, kind):
        self.seq.append((shape, dtype, kind))
        return TorchAlloc().take(shape, dtype, kind)


class SlabAlloc:
    """Serves a recorded allocation sequence from persistent slabs."""

    ALIGN = 256

    def __init__(self, plan: SlabPlan):
        self.seq = list(plan.seq)
        sizes = {"static": 0, "volatile": 0, "status": 0, "host": 0}
        self.offsets = []
        for shape, dtype, kind in self.seq:
            nbytes = max(1, int(np.prod(shape))) * torch.empty((), dtype=dtype).element_size()
            k = "static" if kind == "empty" else kind
            self.offsets.append((k, sizes[k]))
            sizes[k] += -(-nbytes // self.ALIGN) * self.ALIGN
        dev = device()
        self.slabs = {k: torch.zeros(max(v, self.ALIGN), dtype=torch.uint8, device=dev) for k, v in sizes.items()
                      if k != "host"}
        # host staging (segment tables) is pinned, persistent, and allocated before capture:
        # captured H2D memcpy nodes read it at every replay
        self.slabs["host"] = torch.zeros(max(sizes["host"], self.ALIGN), dtype=torch.uint8).pin_memory()
        self.slabs["status"].view(torch.int64).fill_(STATUS_CLEAR)
        self.i = 0

    def reset(self):
        """Per-forward re-initialisation (inside the captured graph)."""
        self.i = 0
        # ONE kernel for both slabs (memset nodes measured 2-3 us slower per C2 epoch than a
        # kernel ahead of the first engine kernel)
        z, st = self.slabs["volatile"], self.slabs["status"]
        check(lib().qg_slab_reset(z.data_ptr(), z.numel() // 8, st.data_ptr(), st.numel() // 8, stream()),
              "qg_slab_reset")

    def take(self, shape, dtype, kind):
        if self.i >= len(self.seq) or self.seq[self.i][0] != shape or self.seq[self.i][1] != dtype:
            raise RuntimeError("allocation sequence diverged from the recorded forward")
        k, off = self.offsets[self.i]
        self.i += 1
        n = int(np.prod(shape))
        nbytes = max(1, n) * torch.empty((), dtype=dtype).element_size()
        return self.slabs[k][off:off + nbytes].view(dtype)[:n].view(shape)


# ------------------------------------------------------------ device helpers
def new_status(n: int = 1) -> torch.Tensor:
    return alloc((n,), torch.int64, "status")


def status_index(status: torch.Tensor) -> int | None:
    """First offending linear index recorded in a status cell, else None."""
    v = int(status[0].item())
    return None if v == STATUS_CLEAR else v


def raise_nonfinite(status: torch.Tensor, cols: int) -> None:
    idx = status_index(status)
    if idx is not None:
        r, c = divmod(idx, cols) if cols else (idx, 0)
        raise DataError(f"non-finite value at ({r}, {c})")


def raise_overflow(flag: torch.Tensor, peak_fn) -> None:
    if int(flag.item()):
        raise ReductionOverflowError(f"reduced value {peak_fn()} does not fit a signed 32-bit output")


def to_device(a, dtype=None) -> torch.Tensor:
    """numpy / list / torch -> contiguous CUDA tensor (single H2D when host)."""
    dev = device()
    if isinstance(a, torch.Tensor):
        t = a.to(dev, non_blocking=True)
    else:
        arr = np.asarray(a)
        if arr.dtype == np.uint32:
            arr = arr.view(np.int32)
        elif arr.dtype == np.uint64:
            arr = arr.view(np.int64)
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(dev, non_blocking=True)
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


def words_to_numpy(t: torch.Tensor) -> np.ndarray:
    """int32 device words -> numpy uint32 (the reference's ``words`` dtype)."""
    return t.detach().cpu().numpy().view(np.uint32)
