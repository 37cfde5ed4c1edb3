"""3D-stacked bit planes packed into u32 words (mirror of bitpack.py).

Layouts are the reference's, verbatim (bitpack.py:3-14), so ``words`` views
are interchangeable with the reference's; the words live in HBM as int32
tensors (``dwords``) and ``words`` is a cached numpy (uint32) view.

A ``BitPlaneStack`` owns ONE contiguous ``(bits, words_per_plane)`` device
tensor; its planes are views into it, which is the layout every kernel reads
(plane p at ``dwords[p]``).
"""

from __future__ import annotations

import struct

import numpy as np
import torch

from . import _native as N
from .errors import DataError, FormatError

WORD_BITS = 32
COLUMN_WISE = "column-wise"
ROW_WISE = "row-wise"

MAGIC = b"QGTC"
VERSION = 1
_HEADER = struct.Struct("<4sHBBIIII")


def orient_id(orientation: str) -> int:
    if orientation == COLUMN_WISE:
        return N.COLUMN_WISE_ID
    if orientation == ROW_WISE:
        return N.ROW_WISE_ID
    raise ValueError(f"unknown orientation {orientation!r}")


def pad8(n: int) -> int:
    """Smallest multiple of 8 >= n (bitpack.py:40-44)."""
    if n < 0:
        raise ValueError("dimension must be non-negative")
    return -(-n // 8) * 8


def pad128(n: int) -> int:
    """Smallest multiple of 128 >= n (bitpack.py:47-51)."""
    if n < 0:
        raise ValueError("dimension must be non-negative")
    return -(-n // 128) * 128


def _pad_to(n: int, multiple: int) -> int:
    if multiple not in (8, 128):
        raise ValueError(f"padding multiple must be 8 or 128, got {multiple}")
    return pad8(n) if multiple == 8 else pad128(n)


def padded_dims(rows: int, cols: int, orientation: str, pad_to: int) -> tuple[int, int]:
    if orientation == COLUMN_WISE:
        return _pad_to(rows, pad_to), pad128(cols)
    return pad128(rows), _pad_to(cols, pad_to)


class PackedBitMatrix:
    """One packed bit plane (bitpack.py:60-99) with device-resident words."""

    def __init__(self, orientation, logical_rows, logical_cols, padded_rows, padded_cols, words):
        if orientation not in (COLUMN_WISE, ROW_WISE):
            raise ValueError(f"unknown orientation {orientation!r}")
        self.orientation = orientation
        self.logical_rows, self.logical_cols = int(logical_rows), int(logical_cols)
        self.padded_rows, self.padded_cols = int(padded_rows), int(padded_cols)
        expect = self.padded_rows * self.padded_cols // WORD_BITS
        if isinstance(words, torch.Tensor):
            t = words.reshape(-1)
            if t.dtype != torch.int32:
                t = t.to(torch.int64).to(torch.int32) if t.dtype != torch.uint32 else t.view(torch.int32)
            self._np = None
        else:
            arr = np.ascontiguousarray(np.asarray(words, dtype=np.uint32)).ravel()
            if len(arr) != expect:
                raise FormatError(f"word count {len(arr)} != padded {self.padded_rows}x"
                                  f"{self.padded_cols}/32 = {expect}")
            self._np = arr
            t = N.to_device(arr)
        if t.numel() != expect:
            raise FormatError(f"word count {t.numel()} != padded {self.padded_rows}x"
                              f"{self.padded_cols}/32 = {expect}")
        self.dwords = t if t.is_cuda else N.to_device(t)
        self._tilemap = None       # scan_zero_tiles cache (bitgemm.py:222-233)
        self._schedule = None      # device zero-tile-jumping schedule + degrees

    @property
    def words(self) -> np.ndarray:
        if self._np is None:
            self._np = N.words_to_numpy(self.dwords)
        return self._np

    @property
    def words2d(self) -> np.ndarray:
        if self.orientation == COLUMN_WISE:
            return self.words.reshape(self.padded_rows, self.padded_cols // WORD_BITS)
        return self.words.reshape(self.padded_cols, self.padded_rows // WORD_BITS)

    def dims(self) -> tuple[int, int, int, int]:
        return self.logical_rows, self.logical_cols, self.padded_rows, self.padded_cols

    def __eq__(self, other):
        return (isinstance(other, PackedBitMatrix) and self.orientation == other.orientation
                and self.dims() == other.dims()
                and bool(torch.equal(self.dwords, other.dwords.to(self.dwords.device))))

    __hash__ = None

    def __repr__(self):
        return (f"PackedBitMatrix({self.orientation}, {self.logical_rows}x{self.logical_cols} "
                f"-> {self.padded_rows}x{self.padded_cols})")


class BitPlaneStack:
    """q identically packed planes (bitpack.py:102-150); one contiguous device block."""

    def __init__(self, bits: int, planes):
        planes = list(planes)
        if bits != len(planes):
            raise ValueError(f"bits={bits} but {len(planes)} planes")
        if not planes:
            raise ValueError("a stack needs at least one plane")
        first = planes[0]
        for p in planes[1:]:
            if p.orientation != first.orientation or p.dims() != first.dims():
                raise ValueError("planes disagree on orientation or padding")
        self.bits = bits
        self.dwords = torch.stack([p.dwords for p in planes]).contiguous()
        self._planes = None
        self._meta = (first.orientation,) + first.dims()

    @classmethod
    def _wrap(cls, orientation, rows, cols, pr, pc, dwords2d: torch.Tensor) -> "BitPlaneStack":
        """Adopt a (bits, words) device tensor without copying."""
        st = cls.__new__(cls)
        st.bits = int(dwords2d.shape[0])
        st.dwords = dwords2d
        st._planes = None
        st._meta = (orientation, int(rows), int(cols), int(pr), int(pc))
        return st

    @property
    def planes(self) -> list[PackedBitMatrix]:
        if self._planes is None:
            o, r, c, pr, pc = self._meta
            self._planes = [PackedBitMatrix(o, r, c, pr, pc, self.dwords[i]) for i in range(self.bits)]
        return self._planes

    @property
    def orientation(self) -> str:
        return self._meta[0]

    @property
    def logical_rows(self) -> int:
        return self._meta[1]

    @property
    def logical_cols(self) -> int:
        return self._meta[2]

    @property
    def padded_rows(self) -> int:
        return self._meta[3]

    @property
    def padded_cols(self) -> int:
        return self._meta[4]

    def dims(self) -> tuple[int, int, int, int]:
        return self._meta[1:]

    def __eq__(self, other):
        return (isinstance(other, BitPlaneStack) and self.bits == other.bits
                and self._meta == other._meta
                and bool(torch.equal(self.dwords, other.dwords.to(self.dwords.device))))

    __hash__ = None

    def __repr__(self):
        return f"BitPlaneStack({self.bits} x {self.orientation} {self.logical_rows}x{self.logical_cols})"


class CodeBackedStack(BitPlaneStack):
    """A stack whose source of truth is a u8 code cache in HBM (the fused GEMM
    epilogues emit codes in the next GEMM's K-major operand layout).  The packed
    plane words -- the reference's ``words`` -- are materialised on first access
    by the bit_qnt kernel (a row-wise packing of M is the column-wise packing of
    M^T, so either code layout serves either orientation)."""

    def __init__(self, orientation, rows, cols, bits, codes: torch.Tensor, ld: int, colmajor: bool, pad_to=8):
        pr, pc = padded_dims(rows, cols, orientation, pad_to)
        self.bits = int(bits)
        self._planes = None
        self._meta = (orientation, int(rows), int(cols), int(pr), int(pc))
        self.codes, self.codes_ld, self.codes_colmajor = codes, int(ld), bool(colmajor)
        self._dwords = None

    @property
    def dwords(self) -> torch.Tensor:
        if self._dwords is None:
            o, rows, cols, pr, pc = self._meta
            # codes viewed as a row-major matrix: M itself, or M^T for col-major codes
            src_rows, src_cols = (cols, rows) if self.codes_colmajor else (rows, cols)
            want_col = (o == COLUMN_WISE) != self.codes_colmajor
            oid = N.COLUMN_WISE_ID if want_col else N.ROW_WISE_ID
            words = torch.empty((self.bits, pr * pc // 32), dtype=torch.int32, device=self.codes.device)
            if words.numel():
                status = N.new_status()
                N.call("qg_quantize_pack", N.ptr(self.codes), N.SRC_U8, src_rows, src_cols, self.codes_ld, 0.0, 1.0,
                       self.bits, oid, 8, N.ptr(words), None, None, None, N.ptr(status), N.stream())
            self._dwords = words
        return self._dwords

    @dwords.setter
    def dwords(self, value):
        self._dwords = value


def stack_code_operand(stack: BitPlaneStack, colmajor: bool, row_sums=None):
    """(u8 codes, ld) of a stack in a K-major operand layout (row-major for a
    left operand, col-major for a right one); reuses a code cache when present.
    ``row_sums`` (int64, zeroed) receives the row code sums when the conversion
    is a row-wise -> row-major transpose."""
    if isinstance(stack, CodeBackedStack) and stack.codes_colmajor == colmajor:
        return stack.codes, stack.codes_ld
    rows, cols, pr, pc = stack.dims()
    ld = pad128(rows if colmajor else cols)
    codes = N.alloc(((cols if colmajor else rows), ld), torch.uint8, "static")
    if rows * cols:
        N.call("qg_planes_to_codes", N.ptr(stack.dwords), stack.bits, rows, cols, pr, pc,
               orient_id(stack.orientation), N.ptr(codes), ld, int(colmajor), N.ptr(row_sums), N.stream())
    return codes, ld


# ------------------------------------------------------------------ packing
def _binary_planes(planes) -> torch.Tensor:
    """(bits, rows, cols) input -> u8 device tensor; non-binary -> DataError."""
    if isinstance(planes, torch.Tensor):
        t = planes.to(N.device())
    else:
        t = N.to_device(np.asarray(planes))
    return t


def _pack_device(t: torch.Tensor, orientation: str, pad_to: int):
    """Pack a (bits, rows, cols) device tensor of 0/1 values; DataError otherwise."""
    bits, rows, cols = t.shape
    pr, pc = padded_dims(rows, cols, orientation, pad_to)
    if t.dtype != torch.uint8:
        bad = (t != 0) & (t != 1)
        if bool(bad.any()):
            p, r, c = (int(v) for v in torch.nonzero(bad)[0])
            raise DataError(f"non-binary entry at ({r}, {c})")
        t = t.to(torch.uint8)
    t = t.contiguous()
    words = torch.empty((bits, pr * pc // 32), dtype=torch.int32, device=t.device)
    if words.numel() == 0:
        return BitPlaneStack._wrap(orientation, rows, cols, pr, pc, words)
    status = N.new_status()
    N.call("qg_pack_planes", N.ptr(t), bits, rows, cols, orient_id(orientation), pad_to, N.ptr(words),
           N.ptr(status), N.stream())
    idx = N.status_index(status)
    if idx is not None:
        rem = idx % (rows * cols)
        raise DataError(f"non-binary entry at ({rem // cols}, {rem % cols})")
    return BitPlaneStack._wrap(orientation, rows, cols, pr, pc, words)


def _as_plane(plane) -> torch.Tensor:
    t = _binary_planes(plane)
    if t.dim() != 2:
        raise ValueError(f"expected a 2-D plane, got ndim={t.dim()}")
    return t.unsqueeze(0)


def pack_colwise(plane, pad_rows_to: int = 8) -> PackedBitMatrix:
    """Column-wise packing of a 0/1 matrix (bitpack.py:169-178)."""
    t = _as_plane(plane)
    _pad_to(0, pad_rows_to)
    return _pack_device(t, COLUMN_WISE, pad_rows_to).planes[0]


def pack_rowwise(plane, pad_cols_to: int = 8) -> PackedBitMatrix:
    """Row-wise packing of a 0/1 matrix (bitpack.py:181-191)."""
    t = _as_plane(plane)
    _pad_to(0, pad_cols_to)
    return _pack_device(t, ROW_WISE, pad_cols_to).planes[0]


def unpack(p: PackedBitMatrix) -> np.ndarray:
    """Logical 0/1 plane (bitpack.py:194-210)."""
    if p.dwords.numel() != p.padded_rows * p.padded_cols // WORD_BITS:
        raise FormatError("word count inconsistent with padded dims")
    return _unpack_device(p.dwords.reshape(1, -1), p.orientation, *p.dims())[0].cpu().numpy()


def _unpack_device(dwords2d, orientation, rows, cols, pr, pc, codes=False):
    bits = dwords2d.shape[0]
    dev = dwords2d.device
    if rows * cols == 0:
        return torch.zeros((rows, cols) if codes else (bits, rows, cols),
                           dtype=torch.int32 if codes else torch.uint8, device=dev)
    if codes:
        out = torch.empty((rows, cols), dtype=torch.int32, device=dev)
        N.call("qg_unpack", N.ptr(dwords2d), bits, rows, cols, pr, pc, orient_id(orientation), None,
               N.ptr(out), N.stream())
        return out
    out = torch.empty((bits, rows, cols), dtype=torch.uint8, device=dev)
    N.call("qg_unpack", N.ptr(dwords2d), bits, rows, cols, pr, pc, orient_id(orientation), N.ptr(out), None,
           N.stream())
    return out


def pack_planes(planes, orientation: str, pad_to: int = 8) -> BitPlaneStack:
    """Pack (bits, rows, cols) planes into a stack (bitpack.py:213-228)."""
    t = _binary_planes(planes)
    if t.dim() != 3:
        raise ValueError(f"expected (bits, rows, cols) planes, got ndim={t.dim()}")
    orient_id(orientation)
    _pad_to(0, pad_to)
    if t.shape[0] == 0:
        raise ValueError("bits=0 but 0 planes")
    return _pack_device(t, orientation, pad_to)


def to_planes(stack: BitPlaneStack) -> np.ndarray:
    """Logical (bits, rows, cols) planes (bitpack.py:231-233)."""
    return _unpack_device(stack.dwords, stack.orientation, *stack.dims()).cpu().numpy()


def stack_codes(stack: BitPlaneStack) -> torch.Tensor:
    """Device int32 codes sum_p plane_p << p of a stack (to_val(to_planes(...)))."""
    return _unpack_device(stack.dwords, stack.orientation, *stack.dims(), codes=True)


def repack(stack: BitPlaneStack, orientation: str, pad_to: int = 8) -> BitPlaneStack:
    """Re-orient a stack (bitpack.py:236-238) with warp bit transposes on the GPU."""
    rows, cols = stack.logical_rows, stack.logical_cols
    pr, pc = padded_dims(rows, cols, orientation, pad_to)
    dst = torch.empty((stack.bits, pr * pc // 32), dtype=torch.int32, device=stack.dwords.device)
    if orientation == stack.orientation:
        # same orientation, new padding: through device logical planes
        planes = _unpack_device(stack.dwords, stack.orientation, *stack.dims())
        return _pack_device(planes, orientation, pad_to)
    N.call("qg_repack", N.ptr(stack.dwords), stack.bits, stack.padded_rows, stack.padded_cols,
           orient_id(stack.orientation), N.ptr(dst), pr, pc, N.stream())
    return BitPlaneStack._wrap(orientation, rows, cols, pr, pc, dst)


def serialize(stack: BitPlaneStack) -> bytes:
    """Byte-exact image of a stack (bitpack.py:241-256)."""
    orient = 0 if stack.orientation == COLUMN_WISE else 1
    header = _HEADER.pack(MAGIC, VERSION, orient, stack.bits, stack.logical_rows, stack.logical_cols,
                          stack.padded_rows, stack.padded_cols)
    return header + stack.dwords.cpu().numpy().astype("<i4").tobytes()


def deserialize(data: bytes) -> BitPlaneStack:
    """Inverse of serialize (bitpack.py:259-285); one H2D of the plane block."""
    if len(data) < _HEADER.size:
        raise FormatError("payload shorter than header")
    magic, version, orient, bits, lr, lc, pr, pc = _HEADER.unpack_from(data)
    if magic != MAGIC:
        raise FormatError(f"bad magic {magic!r}")
    if version != VERSION:
        raise FormatError(f"unsupported version {version}")
    if orient not in (0, 1):
        raise FormatError(f"bad orientation byte {orient}")
    if not 1 <= bits <= 64:
        raise FormatError(f"bad plane count {bits}")
    wpp = pr * pc // WORD_BITS
    expect = _HEADER.size + bits * wpp * 4
    if len(data) != expect:
        raise FormatError(f"payload length {len(data)} != expected {expect}")
    raw = np.frombuffer(data, dtype="<i4", count=bits * wpp, offset=_HEADER.size).reshape(bits, wpp)
    orientation = COLUMN_WISE if orient == 0 else ROW_WISE
    return BitPlaneStack._wrap(orientation, lr, lc, pr, pc, N.to_device(raw))
