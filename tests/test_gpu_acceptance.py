"""The reference's acceptance criteria (pkg/tests/test_acceptance.py), run against the
CUDA path: every result exact against numpy int64 arithmetic or the CPU oracle."""

import numpy as np
import pytest

import paper_2111_09547_b200 as bg
from oracle import qgtc_oracle as O

pytestmark = pytest.mark.gpu


def quantized_stack(rng, rows, cols, bits, orientation):
    vals = rng.integers(0, 2 ** bits, (rows, cols))
    qm = bg.quantize_matrix(vals.astype(np.float64), bg.QuantParams(0.0, float(2 ** bits), bits))
    return bg.pack_planes(bg.bit_decompose(qm), orientation), qm.values.astype(np.int64)


def test_gemm_oracle_equivalence_200_instances():
    """test_acceptance.py:63-76: 200 random shapes and bit widths, exact."""
    rng = np.random.default_rng(2024)
    for _ in range(200):
        m, k, n = (int(v) for v in rng.integers(1, 257, 3))
        s, t = (int(v) for v in rng.integers(1, 9, 2))
        xs, xv = quantized_stack(rng, m, k, s, bg.COLUMN_WISE)
        ws, wv = quantized_stack(rng, k, n, t, bg.ROW_WISE)
        acc = bg.gemm_sbit_by_tbit(xs, ws, "int32")
        np.testing.assert_array_equal(acc, (xv @ wv).astype(np.int32))


def test_scalar_composition_exhaustive():
    """test_acceptance.py:79-101: every a*b for s, t <= 4 through the bit-plane GEMM."""
    for s in range(1, 5):
        for t in range(1, 5):
            a = np.arange(2 ** s, dtype=np.float64)[:, None]          # one row per value of a
            b = np.arange(2 ** t, dtype=np.float64)[None, :]          # one column per value of b
            qa = bg.quantize_matrix(a, bg.QuantParams(0.0, float(2 ** s), s))
            qb = bg.quantize_matrix(b, bg.QuantParams(0.0, float(2 ** t), t))
            xs = bg.pack_planes(bg.bit_decompose(qa), bg.COLUMN_WISE)
            ws = bg.pack_planes(bg.bit_decompose(qb), bg.ROW_WISE)
            got = bg.gemm_sbit_by_tbit(xs, ws, "int32")
            np.testing.assert_array_equal(got, (a @ b).astype(np.int32))


def test_packing_laws():
    """test_acceptance.py:104-128: pack/unpack round trips + word layout probes."""
    rng = np.random.default_rng(7)
    for orientation in (bg.COLUMN_WISE, bg.ROW_WISE):
        pack = bg.pack_colwise if orientation == bg.COLUMN_WISE else bg.pack_rowwise
        for _ in range(100):
            r, c = (int(v) for v in rng.integers(1, 301, 2))
            plane = (rng.uniform(0, 1, (r, c)) < 0.5).astype(np.uint8)
            p = pack(plane)
            np.testing.assert_array_equal(bg.unpack(p), plane)
            o = O.COL if orientation == bg.COLUMN_WISE else O.ROW
            w, pr, pc = O.pack_words(plane, o, 8)
            np.testing.assert_array_equal(p.words, w)
    stack, _ = quantized_stack(rng, 50, 300, 3, bg.COLUMN_WISE)
    data = bg.serialize(stack)
    assert bg.serialize(bg.deserialize(data)) == data


def test_zero_tile_jumping():
    """test_acceptance.py:139-169: jump on/off identical, skip counts exact."""
    rng = np.random.default_rng(11)
    for _ in range(60):
        m, k, n = int(rng.integers(1, 200)), int(rng.integers(1, 520)), int(rng.integers(1, 24))
        s = int(rng.integers(1, 5))
        dense = (rng.uniform(0, 1, (m, k)) < 0.02).astype(np.uint8)
        a = bg.pack_colwise(dense)
        stack, sv = quantized_stack(rng, k, n, s, bg.ROW_WISE)
        with_jump = bg.bmm_1bit_by_nbit(a, stack, jump=True)
        skipped = bg.op_counters().tiles_skipped
        without = bg.bmm_1bit_by_nbit(a, stack, jump=False)
        for p, (x, y) in enumerate(zip(with_jump, without)):
            np.testing.assert_array_equal(x, y)
            np.testing.assert_array_equal(x, dense.astype(np.int64) @ ((sv >> p) & 1))
        flags = O.zero_tile_flags(a.words, a.padded_rows, a.padded_cols)
        assert skipped == int(flags.sum())


def test_nonzero_tile_reuse():
    """test_acceptance.py:172-187: O(1) adjacency fetches under cross-tile reduction."""
    rng = np.random.default_rng(13)
    a = bg.pack_colwise(np.ones((64, 256), dtype=np.uint8))
    nz = int((~bg.scan_zero_tiles(a).flags).sum())
    assert nz == (64 // 8) * (256 // 128)
    for s in (1, 2, 4, 8):
        stack, _ = quantized_stack(rng, 256, 16, s, bg.ROW_WISE)
        out_tile = bg.bmm_1bit_by_nbit(a, stack, reuse=bg.CROSS_TILE)
        assert bg.op_counters().tile_fetch_count == nz
        out_bit = bg.bmm_1bit_by_nbit(a, stack, reuse=bg.CROSS_BIT)
        assert bg.op_counters().tile_fetch_count == s * nz
        for x, y in zip(out_tile, out_bit):
            np.testing.assert_array_equal(x, y)


def test_work_scales_with_bit_widths():
    """test_acceptance.py:194-204: word_and_popcount_count proportional to s*t."""
    counts = {}
    for s in (1, 2, 4, 8):
        for t in (1, 2, 4, 8):
            xs = bg.pack_planes(np.ones((s, 40, 200), dtype=np.uint8), bg.COLUMN_WISE)
            ws = bg.pack_planes(np.ones((t, 200, 24), dtype=np.uint8), bg.ROW_WISE)
            acc = bg.gemm_sbit_by_tbit(xs, ws, "int32")
            assert int(acc[0, 0]) == ((1 << s) - 1) * ((1 << t) - 1) * 200
            counts[s, t] = bg.op_counters().word_and_popcount_count
    base = counts[1, 1]
    assert base > 0 and all(v == s * t * base for (s, t), v in counts.items())
