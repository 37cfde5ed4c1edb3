"""CPU oracle for the QGTC hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference ``bitgnn`` algorithm for
the hot path (quantize -> bit planes -> packed words -> bit-serial AND+popcount
GEMMs with zero-tile jumping -> fp64 epilogue -> GCN/GIN layer forward).  It is
written independently of the reference sources; every function cites the
reference ``file:line`` whose behaviour it restates (paths are relative to
``/root/reference/pkg/src/bitgnn``).

Who may use it: ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg -- only as the checker or as the
timed CPU baseline, never as the product path.  The product package
(``paper_2111_09547_b200``) never imports this module.

Pinning: the restatement is checked against golden vectors produced by the
real reference (``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``) in
``tests/test_oracle_golden.py``.

Layouts (bitpack.py:3-14): column-wise words ``[padded_rows][padded_cols/32]``
hold 32 consecutive columns of one row; row-wise words
``[padded_cols][padded_rows/32]`` hold 32 consecutive rows of one column; bit j
of word w is element ``32w + j``.
"""

from __future__ import annotations

import math

import numpy as np

COL = "column-wise"
ROW = "row-wise"
TILE_R, TILE_C, TILE_KW = 8, 8, 4          # bitgemm.py:39-42
INT32_MAX, INT32_MIN = 2 ** 31 - 1, -(2 ** 31)


# ---------------------------------------------------------------- quantize --
def grid_scale(amin: float, amax: float, bits: int) -> float:
    """scale = (alpha_max - alpha_min) / 2**bits in fp64 (quantize.py:41)."""
    return (amax - amin) / (1 << bits)


def quantize_codes(m, amin: float, amax: float, bits: int) -> np.ndarray:
    """clip(floor((a - amin) / scale), 0, 2**bits - 1) in fp64 (quantize.py:93-105)."""
    a = np.asarray(m, dtype=np.float64)
    scale = grid_scale(amin, amax, bits)
    v = np.floor((a - amin) / scale)
    return np.clip(v, 0, (1 << bits) - 1).astype(np.uint8)


def first_nonfinite(m):
    """(r, c) of the first non-finite entry in row-major order, else None (quantize.py:98-101)."""
    a = np.asarray(m, dtype=np.float64)
    bad = np.argwhere(~np.isfinite(a))
    return None if len(bad) == 0 else (int(bad[0][0]), int(bad[0][1]))


def planes_of(codes: np.ndarray, bits: int) -> np.ndarray:
    """(bits, rows, cols) 0/1 planes, plane i = bit i (quantize.py:108-112)."""
    c = np.asarray(codes, dtype=np.uint8)
    return np.stack([(c >> i) & 1 for i in range(bits)]).astype(np.uint8)


def codes_of(planes: np.ndarray) -> np.ndarray:
    """sum_i 2**i * plane_i as int32 (quantize.py:115-129)."""
    p = np.asarray(planes, dtype=np.int64)
    w = (1 << np.arange(p.shape[0], dtype=np.int64))[:, None, None]
    return (p * w).sum(axis=0).astype(np.int32)


# ----------------------------------------------------------------- packing --
def pad_up(n: int, mult: int) -> int:
    """Ceil to a multiple of 8 or 128 (bitpack.py:40-57)."""
    return -(-n // mult) * mult


def _bits_to_words(bits2d: np.ndarray) -> np.ndarray:
    # little-endian bit order inside each u32 word (bitpack.py:10-11, 163-166)
    return np.packbits(bits2d, axis=1, bitorder="little").view("<u4").astype(np.uint32)


def pack_words(plane, orientation: str, pad_to: int = 8):
    """Pack one 0/1 plane; returns (words_flat, padded_rows, padded_cols).

    Column-wise: rows pad ``pad_to``, cols pad 128 (bitpack.py:169-178).
    Row-wise: rows pad 128, cols pad ``pad_to`` (bitpack.py:181-191).
    """
    a = np.asarray(plane, dtype=np.uint8)
    rows, cols = a.shape
    if orientation == COL:
        pr, pc = pad_up(rows, pad_to), pad_up(cols, 128)
        buf = np.zeros((pr, pc), np.uint8)
        buf[:rows, :cols] = a
        return _bits_to_words(buf).ravel(), pr, pc
    pr, pc = pad_up(rows, 128), pad_up(cols, pad_to)
    buf = np.zeros((pc, pr), np.uint8)
    buf[:cols, :rows] = a.T
    return _bits_to_words(buf).ravel(), pr, pc


def pack_stack(planes, orientation: str, pad_to: int = 8):
    """Pack (bits, rows, cols) planes -> ((bits, words) array, pr, pc) (bitpack.py:213-228)."""
    out = [pack_words(p, orientation, pad_to) for p in np.asarray(planes, np.uint8)]
    return np.stack([o[0] for o in out]), out[0][1], out[0][2]


def words2d(words, orientation: str, pr: int, pc: int) -> np.ndarray:
    """Row view of a packed plane (bitpack.py:83-88)."""
    w = np.asarray(words, dtype=np.uint32)
    return w.reshape(pr, pc // 32) if orientation == COL else w.reshape(pc, pr // 32)


def unpack_words(words, orientation: str, rows: int, cols: int, pr: int, pc: int) -> np.ndarray:
    """Logical 0/1 plane from packed words (bitpack.py:194-210)."""
    w2 = words2d(words, orientation, pr, pc)
    bits = np.unpackbits(w2.astype("<u4").view(np.uint8), axis=1, bitorder="little")
    if orientation == COL:
        return bits[:rows, :cols]
    return bits.T[:rows, :cols]


# -------------------------------------------------------------- tile scan --
def popcount_u32(v) -> np.ndarray:
    """Per-word popcount via byte table (same values as bitgemm.py:48-60)."""
    v = np.ascontiguousarray(np.asarray(v, dtype=np.uint32))
    table = np.array([bin(i).count("1") for i in range(256)], dtype=np.uint32)
    return table[v.view(np.uint8)].reshape(v.shape + (4,)).sum(axis=-1, dtype=np.uint32)


def zero_tile_flags(col_words, pr: int, pc: int) -> np.ndarray:
    """True for all-zero 8x128 tiles of a column-wise plane (bitgemm.py:214-233)."""
    rt, ct = pr // TILE_R, pc // 128
    if rt == 0 or ct == 0:
        return np.zeros((rt, ct), dtype=bool)
    w = words2d(col_words, COL, pr, pc).reshape(rt, TILE_R, ct, TILE_KW)
    return np.bitwise_or.reduce(np.bitwise_or.reduce(w, axis=3), axis=1) == 0


def row_degrees(col_words, pr: int, pc: int, rows: int) -> np.ndarray:
    """Out-degree per row = popcount row sums, int64 (graph.py:292-295)."""
    return popcount_u32(words2d(col_words, COL, pr, pc)).sum(axis=1, dtype=np.int64)[:rows]


# ------------------------------------------------------------ bit GEMMs --
def _active_rows(flags_col: np.ndarray, jump: bool, rt: int):
    """Rows touched by one 128-bit tile column (bitgemm.py:262-279)."""
    if not jump:
        return None
    nz = np.nonzero(~flags_col)[0]
    if len(nz) == rt:
        return None
    return (nz[:, None] * TILE_R + np.arange(TILE_R)).ravel()


def _and_popc(a_blk: np.ndarray, b_blk: np.ndarray) -> np.ndarray:
    """(R,4)x(C,4) words -> (R,C) sum of popcount(a & b): one 128-bit K slice (bitgemm.py:256-259)."""
    return popcount_u32(a_blk[:, None, :] & b_blk[None, :, :]).sum(axis=2, dtype=np.uint32)


def bitserial_product(a_w2: np.ndarray, b_w2: np.ndarray, flags, jump: bool) -> np.ndarray:
    """uint32 (Mp, Np) = A_plane @ B_plane over packed words, tile column by tile column,
    skipping all-zero 8x128 A tiles when ``jump`` (bitgemm.py:337-362)."""
    mp, kw = a_w2.shape
    acc = np.zeros((mp, b_w2.shape[0]), dtype=np.uint32)
    rt = mp // TILE_R
    for tj in range(kw // TILE_KW):
        sl = slice(tj * TILE_KW, tj * TILE_KW + TILE_KW)
        idx = _active_rows(flags[:, tj], jump, rt) if flags is not None else None
        if idx is None:
            acc += _and_popc(a_w2[:, sl], b_w2[:, sl])
        elif len(idx):
            acc[idx] += _and_popc(a_w2[idx, sl], b_w2[:, sl])
    return acc


def bmm_planes(a_words, a_dims, x_stack, x_dims, *, jump=True):
    """Per-plane A(1-bit, column-wise) @ X_p (row-wise): list of int32 (M, N) (bitgemm.py:306-371).

    a_dims = (rows, cols, pr, pc); x_dims = (rows, cols, pr, pc) of each X plane.
    """
    ml, _, mp, apc = a_dims
    _, nl, xpr, xpc = x_dims
    a2 = words2d(a_words, COL, mp, apc)
    flags = zero_tile_flags(a_words, mp, apc)
    out = []
    for p in range(len(x_stack)):
        b2 = words2d(x_stack[p], ROW, xpr, xpc)
        out.append(bitserial_product(a2, b2, flags, jump)[:ml, :nl].astype(np.int32))
    return out


def narrow_int32(total: np.ndarray) -> np.ndarray:
    """int64 -> int32; None signals overflow (bitgemm.py:282-288)."""
    if total.size and (total.max() > INT32_MAX or total.min() < INT32_MIN):
        return None
    return total.astype(np.int32)


def shift_reduce(plane_accs) -> np.ndarray:
    """sum_p acc_p << p in int64 (bitgemm.py:291-298); caller narrows."""
    total = np.zeros(np.asarray(plane_accs[0]).shape, dtype=np.int64)
    for p, acc in enumerate(plane_accs):
        total += np.asarray(acc, dtype=np.int64) << p
    return total


def gemm_planes(x_stack, x_dims, w_stack, w_dims, *, jump=True) -> np.ndarray:
    """int64 (M, N) = sum_{i,j} (X_i @ W_j) << (i+j); X column-wise, W row-wise (bitgemm.py:374-453)."""
    ml, _, mp, xpc = x_dims
    _, nl, wpr, wpc = w_dims
    s, t = len(x_stack), len(w_stack)
    groups = np.zeros((s + t - 1, mp, wpc), dtype=np.int64)
    w2 = [words2d(w, ROW, wpr, wpc) for w in w_stack]
    for i in range(s):
        x2 = words2d(x_stack[i], COL, mp, xpc)
        flags = zero_tile_flags(x_stack[i], mp, xpc)
        for j in range(t):
            groups[i + j] += bitserial_product(x2, w2[j], flags, jump)
    total = np.zeros((mp, wpc), dtype=np.int64)
    for b in range(s + t - 1):
        total += groups[b] << b
    return total[:ml, :nl]


def counters_bmm(flags: np.ndarray, s: int, n_chunks: int, *, jump=True, cross_tile=True) -> dict:
    """Closed forms of the reference counters for bmm (bitgemm.py:335-370)."""
    total = flags.size
    nz = int((~flags).sum()) if jump else total
    mma = s * nz * n_chunks
    return dict(tile_mma_count=mma, tile_fetch_count=nz if cross_tile else s * nz,
                tiles_skipped=int(flags.sum()) if jump else 0,
                word_and_popcount_count=256 * mma, tiles_total=total)


def counters_gemm(plane_flags, t: int, n_chunks: int, *, jump=True, cross_tile=True) -> dict:
    """Closed forms of the reference counters for the s x t GEMM (bitgemm.py:409-461)."""
    nzs = [int((~f).sum()) if jump else f.size for f in plane_flags]
    mma = t * sum(nzs) * n_chunks
    return dict(tile_mma_count=mma, tile_fetch_count=sum(nzs) if cross_tile else t * sum(nzs),
                tiles_skipped=sum(int(f.sum()) for f in plane_flags) if jump else 0,
                word_and_popcount_count=256 * mma,
                tiles_total=sum(f.size for f in plane_flags))


# --------------------------------------------------------------- epilogue --
def dequantize(acc, lhs=None, rhs=None, row_sums=None, col_sums=None, inner_dim=0) -> np.ndarray:
    """fp64 dequantization with the contract term grouping (bitgemm.py:156-179).

    ``lhs``/``rhs`` are (alpha_min, scale) tuples or None (exact integer operand).
    """
    ama, sa = lhs if lhs is not None else (0.0, 1.0)
    amb, sb = rhs if rhs is not None else (0.0, 1.0)
    real = (sa * sb) * np.asarray(acc).astype(np.float64)
    if amb != 0.0:
        real = real + (sa * amb) * np.asarray(row_sums, dtype=np.float64)[:, None]
    if ama != 0.0:
        real = real + (sb * ama) * np.asarray(col_sums, dtype=np.float64)[None, :]
    if ama != 0.0 and amb != 0.0:
        real = real + (float(inner_dim) * ama) * amb
    return real


def finish(real, bias=None, bn=None, kind="none") -> np.ndarray:
    """bias -> batch-norm -> relu/tanh in fp64 (bitgemm.py:192-207).

    ``bn`` = (mean, var, gamma, beta, eps) or None.
    """
    if bias is not None:
        real = real + np.asarray(bias, dtype=np.float64)[None, :]
    if bn is not None:
        mean, var, gamma, beta, eps = bn
        real = ((real - mean[None, :]) / np.sqrt(var + eps)[None, :]) * gamma[None, :] + beta[None, :]
    if kind == "relu":
        real = np.maximum(real, 0.0)
    elif kind == "tanh":
        real = np.tanh(real).astype(np.float32).astype(np.float64)
    return real


# ---------------------------------------------------------- layer forward --
def _grid(p):
    return (p.alpha_min, p.scale) if p is not None else None


def _bn_tuple(bn):
    return None if bn is None else (bn.mean, bn.var, bn.gamma, bn.beta, bn.eps)


def _requant(real, params, orientation):
    codes = quantize_codes(real, params.alpha_min, params.alpha_max, params.bits)
    words, pr, pc = pack_stack(planes_of(codes, params.bits), orientation, 8)
    return codes, words, (codes.shape[0], codes.shape[1], pr, pc)


def model_forward(adj_words, adj_dims, feat_codes, x_params, layers, *, jump=True):
    """Quantized GCN/GIN forward over packed operands (engine.py:209-332).

    ``layers`` are objects with the reference LayerConfig fields.  Follows
    ``_aggregate_then_update`` (engine.py:235-276) and
    ``_update_then_aggregate`` (engine.py:279-317) step for step: every
    product runs bit-serially on packed words, every requantization goes
    through fp64 ``quantize_codes``.  Returns fp64 logits.
    """
    n = adj_dims[0]
    deg = row_degrees(adj_words, adj_dims[2], adj_dims[3], n)
    codes = np.asarray(feat_codes, dtype=np.uint8)
    params = x_params
    out = None
    for li, ly in enumerate(layers):
        last = li == len(layers) - 1
        wq = quantize_codes(ly.weight, ly.weight_params.alpha_min, ly.weight_params.alpha_max,
                            ly.weight_params.bits)
        w_cols = wq.sum(axis=0, dtype=np.int64)
        w_words, wpr, wpc = pack_stack(planes_of(wq, ly.weight_params.bits), ROW,
                                       128 if ly.output_mode == "bitplanes" else 8)
        w_dims = (wq.shape[0], wq.shape[1], wpr, wpc)
        if ly.order == "aggregate-then-update":
            xw, xpr, xpc = pack_stack(planes_of(codes, params.bits), ROW, 8)
            accs = bmm_planes(adj_words, adj_dims, xw, (n, codes.shape[1], xpr, xpc), jump=jump)
            agg = narrow_int32(shift_reduce(accs))
            real = dequantize(agg, None, _grid(params), deg, None, n)
            mid, mw, mdims = _requant(real, ly.mid_params, COL)
            acc = narrow_int32(gemm_planes(mw, mdims, w_words, w_dims, jump=jump))
            real = dequantize(acc, _grid(ly.mid_params), _grid(ly.weight_params),
                              mid.sum(axis=1, dtype=np.int64), w_cols, ly.in_dim)
            real = finish(real, ly.bias, _bn_tuple(ly.bn), ly.activation)
        else:
            xw, xpr, xpc = pack_stack(planes_of(codes, params.bits), COL, 8)
            acc = narrow_int32(gemm_planes(xw, (n, codes.shape[1], xpr, xpc), w_words, w_dims,
                                           jump=jump))
            real = dequantize(acc, _grid(params), _grid(ly.weight_params),
                              codes.sum(axis=1, dtype=np.int64), w_cols, ly.in_dim)
            real = finish(real, ly.bias)
            mid, mw, mdims = _requant(real, ly.mid_params, ROW)
            accs = bmm_planes(adj_words, adj_dims, mw, mdims, jump=jump)
            agg = narrow_int32(shift_reduce(accs))
            real = dequantize(agg, None, _grid(ly.mid_params), deg, None, n)
            real = finish(real, None, _bn_tuple(ly.bn), ly.activation)
        if last:
            out = real
        else:
            codes = quantize_codes(real, ly.out_params.alpha_min, ly.out_params.alpha_max,
                                   ly.out_params.bits)
            params = ly.out_params
    return out


def dense_int_forward(dense_a, feat_codes, x_params, layers) -> np.ndarray:
    """Independent check of ``model_forward``: int64 matmuls instead of bit-serial
    products, same fp64 epilogue expressions (mirrors the reference test oracle
    ``tests/oracles.py:107-146``)."""
    a = np.asarray(dense_a, dtype=np.int64)
    deg = a.sum(axis=1)
    h = np.asarray(feat_codes, dtype=np.int64)
    params = x_params
    out = None
    for li, ly in enumerate(layers):
        w = quantize_codes(ly.weight, ly.weight_params.alpha_min, ly.weight_params.alpha_max,
                           ly.weight_params.bits).astype(np.int64)
        if ly.order == "aggregate-then-update":
            real = dequantize(a @ h, None, _grid(params), deg, None, a.shape[1])
            mid = quantize_codes(real, ly.mid_params.alpha_min, ly.mid_params.alpha_max,
                                 ly.mid_params.bits).astype(np.int64)
            real = dequantize(mid @ w, _grid(ly.mid_params), _grid(ly.weight_params),
                              mid.sum(axis=1), w.sum(axis=0), ly.in_dim)
            real = finish(real, ly.bias, _bn_tuple(ly.bn), ly.activation)
        else:
            real = dequantize(h @ w, _grid(params), _grid(ly.weight_params), h.sum(axis=1),
                              w.sum(axis=0), ly.in_dim)
            real = finish(real, ly.bias)
            mid = quantize_codes(real, ly.mid_params.alpha_min, ly.mid_params.alpha_max,
                                 ly.mid_params.bits).astype(np.int64)
            real = dequantize(a @ mid, None, _grid(ly.mid_params), deg, None, a.shape[1])
            real = finish(real, None, _bn_tuple(ly.bn), ly.activation)
        if li == len(layers) - 1:
            out = real
        else:
            h = quantize_codes(real, ly.out_params.alpha_min, ly.out_params.alpha_max,
                               ly.out_params.bits).astype(np.int64)
            params = ly.out_params
    return out


def scalar_quantize(alpha: float, amin: float, amax: float, bits: int) -> int:
    """Pure-Python scalar quantizer (quantize.py:83-90) for small KAT checks."""
    v = math.floor((alpha - amin) / grid_scale(amin, amax, bits))
    return min(max(v, 0), (1 << bits) - 1)
