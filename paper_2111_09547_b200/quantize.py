"""Eq.2 uniform quantization and bit planes (mirror of quantize.py).

``QuantParams`` / ``quantize_scalar`` are host-side scalar definitions (as in
the reference, quantize.py:22-90).  Matrix quantization runs on the GPU
through ``qg_quantize_pack``; ``QuantMatrix`` keeps its codes device-resident
and exposes ``values`` as a cached numpy view.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N

MAX_BITS = 8


@dataclass(frozen=True)
class QuantParams:
    """Per-tensor grid over [alpha_min, alpha_max) (quantize.py:22-50)."""

    alpha_min: float
    alpha_max: float
    bits: int
    scale: float = field(init=False)

    def __post_init__(self):
        if not 1 <= self.bits <= MAX_BITS:
            raise ValueError(f"bits must be in [1, {MAX_BITS}], got {self.bits}")
        if not (math.isfinite(self.alpha_min) and math.isfinite(self.alpha_max)):
            raise ValueError("alpha bounds must be finite")
        if not self.alpha_max > self.alpha_min:
            raise ValueError(
                f"alpha_max ({self.alpha_max}) must exceed alpha_min ({self.alpha_min})")
        object.__setattr__(self, "scale", (self.alpha_max - self.alpha_min) / (1 << self.bits))

    @property
    def max_value(self) -> int:
        return (1 << self.bits) - 1

    def dequantize_offset_scale(self) -> tuple[float, float]:
        return self.alpha_min, self.scale


class QuantMatrix:
    """Dense q-bit codes (quantize.py:53-80); device-resident ``dvalues`` (u8)."""

    def __init__(self, rows: int, cols: int, values, bits: int):
        if not 1 <= bits <= MAX_BITS:
            raise ValueError(f"bits must be in [1, {MAX_BITS}], got {bits}")
        self.rows, self.cols, self.bits = int(rows), int(cols), int(bits)
        if isinstance(values, torch.Tensor) and values.is_cuda:
            t = values
        else:
            arr = np.asarray(values)
            if arr.shape != (self.rows, self.cols):
                raise ValueError("values shape does not match declared dims")
            if arr.size and (arr.min() < 0 or arr.max() > (1 << bits) - 1):
                raise ValueError(f"values exceed the {bits}-bit range")
            t = N.to_device(arr.astype(np.uint8))
        if tuple(t.shape) != (self.rows, self.cols):
            raise ValueError("values shape does not match declared dims")
        self.dvalues = t.to(torch.uint8).contiguous()
        self._np = None
        self._planes = None  # cached packed planes from the fused kernel, keyed by layout

    @property
    def values(self) -> np.ndarray:
        if self._np is None:
            self._np = self.dvalues.cpu().numpy()
        return self._np

    def __eq__(self, other):
        return (isinstance(other, QuantMatrix) and self.rows == other.rows
                and self.cols == other.cols and self.bits == other.bits
                and bool(torch.equal(self.dvalues, other.dvalues.to(self.dvalues.device))))

    __hash__ = None


def quantize_scalar(alpha: float, p: QuantParams) -> int:
    """One real value onto the grid (quantize.py:83-90).  Scalar host helper."""
    v = math.floor((alpha - p.alpha_min) / p.scale)
    return min(max(v, 0), p.max_value)


def _real_source(m) -> tuple[torch.Tensor, int]:
    """Real matrix -> (2-D CUDA tensor, source kind)."""
    if isinstance(m, torch.Tensor):
        t = m.to(N.device())
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
    else:
        a = np.asarray(m, dtype=np.float64)
        t = N.to_device(a)
    if t.dim() != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={t.dim()}")
    t = t.contiguous()
    return t, (N.SRC_F32 if t.dtype == torch.float32 else N.SRC_F64)


def quantize_pack_device(m, p: QuantParams, orientation_id: int, pad_to: int, *, codes=False,
                         row_sums=False, col_sums=False, check=True):
    """Fused bit_qnt on the GPU: returns a dict of device tensors.

    planes (bits, words), optional codes u8, row/col sums int64 and the status
    cell (non-finite index).  With ``check`` the status is read (one sync) and
    DataError raised like quantize_matrix (quantize.py:98-101).
    """
    t, kind = _real_source(m)
    rows, cols = t.shape
    if orientation_id == N.COLUMN_WISE_ID:
        pr, pc = -(-rows // pad_to) * pad_to, -(-cols // 128) * 128
    else:
        pr, pc = -(-rows // 128) * 128, -(-cols // pad_to) * pad_to
    dev = t.device
    planes = torch.empty((p.bits, pr * pc // 32), dtype=torch.int32, device=dev)
    out = {"planes": planes, "pr": pr, "pc": pc, "rows": rows, "cols": cols}
    out["codes"] = torch.empty((rows, cols), dtype=torch.uint8, device=dev) if codes else None
    out["row_sums"] = torch.zeros(rows, dtype=torch.int64, device=dev) if row_sums else None
    out["col_sums"] = torch.zeros(cols, dtype=torch.int64, device=dev) if col_sums else None
    status = N.new_status()
    out["status"] = status
    N.call("qg_quantize_pack", N.ptr(t), kind, rows, cols, cols, float(p.alpha_min), float(p.scale),
           p.bits, orientation_id, pad_to, N.ptr(planes), N.ptr(out["codes"]), N.ptr(out["row_sums"]),
           N.ptr(out["col_sums"]), N.ptr(status), N.stream())
    if check:
        N.raise_nonfinite(status, cols)
    return out


def quantize_matrix(m, p: QuantParams) -> QuantMatrix:
    """Elementwise Eq.2 quantization on the GPU (quantize.py:93-105)."""
    r = quantize_pack_device(m, p, N.COLUMN_WISE_ID, 8, codes=True)
    qm = QuantMatrix(r["rows"], r["cols"], r["codes"], p.bits)
    qm._planes = ("column-wise", 8, r["planes"], r["pr"], r["pc"])
    return qm


def bit_decompose(qm: QuantMatrix) -> np.ndarray:
    """(bits, rows, cols) 0/1 planes, plane i = bit i (quantize.py:108-112)."""
    shifts = torch.arange(qm.bits, dtype=torch.uint8, device=qm.dvalues.device)
    planes = (qm.dvalues.unsqueeze(0) >> shifts[:, None, None]) & 1
    return planes.cpu().numpy()


def to_val(planes) -> np.ndarray:
    """Recompose planes into int32 codes (quantize.py:115-129)."""
    if isinstance(planes, torch.Tensor):
        p = planes.to(N.device())
    else:
        try:
            arr = np.asarray(planes, dtype=np.uint8)
        except ValueError as exc:
            raise ValueError(f"inconsistent plane dims: {exc}") from None
        p = None
        if arr.ndim != 3:
            raise ValueError(f"expected (bits, rows, cols) planes, got ndim={arr.ndim}")
        p = N.to_device(arr)
    if p.dim() != 3:
        raise ValueError(f"expected (bits, rows, cols) planes, got ndim={p.dim()}")
    if not 1 <= p.shape[0] <= 64:
        raise ValueError(f"unsupported plane count {p.shape[0]}")
    w = torch.ones(p.shape[0], dtype=torch.int64, device=p.device) << torch.arange(
        p.shape[0], dtype=torch.int64, device=p.device)
    return (p.to(torch.int64) * w[:, None, None]).sum(dim=0).to(torch.int32).cpu().numpy()

