"""Pin the CPU oracle (oracle/qgtc_oracle.py) to the reference's golden vectors.

CPU only.  The oracle is the checker for every GPU parity test, so it must
first agree with the real reference bit for bit on the committed fixtures
(tests/golden/make_golden.py ran the reference to produce them).
"""

import numpy as np
import pytest

from golden_io import load, model_case
from oracle import qgtc_oracle as O


def test_quantize_kats_and_matrices():
    d = load("quantize")
    for x, (lo, hi, bits), want in zip(d["kat_in"], d["kat_grid"], d["kat_out"]):
        assert O.scalar_quantize(float(x), lo, hi, int(bits)) == want
        assert O.quantize_codes([[x]], lo, hi, int(bits))[0, 0] == want
    for i in range(int(d["n_matrix"])):
        lo, hi, bits = d[f"m{i}_grid"]
        got = O.quantize_codes(d[f"m{i}_in"], lo, hi, int(bits))
        np.testing.assert_array_equal(got, d[f"m{i}_codes"])


def test_quantize_reference_kats_literal():
    # test_quantize.py:43-54 of the reference: 5.7 -> 5, 0.49 -> 2, alpha_max -> 7
    assert O.scalar_quantize(5.7, 0.0, 8.0, 3) == 5
    assert O.scalar_quantize(0.49, -1.0, 1.0, 2) == 2
    assert O.scalar_quantize(1.0, -1.0, 1.0, 3) == 7
    assert O.scalar_quantize(-5.0, 0.0, 1.0, 3) == 0


def test_pack_words_repack_and_serialize_layout():
    d = load("pack")
    for i in range(int(d["n"])):
        planes = d[f"c{i}_planes"]
        orient_i, pad, pr, pc = (int(v) for v in d[f"c{i}_meta"])
        orient = O.COL if orient_i == 0 else O.ROW
        words, gpr, gpc = O.pack_stack(planes, orient, pad)
        assert (gpr, gpc) == (pr, pc)
        np.testing.assert_array_equal(words, d[f"c{i}_words"])
        back = np.stack([O.unpack_words(w, orient, planes.shape[1], planes.shape[2], pr, pc)
                         for w in words])
        np.testing.assert_array_equal(back, planes)
        other = O.ROW if orient == O.COL else O.COL
        rw, rpr, rpc = O.pack_stack(planes, other, 8)
        assert (rpr, rpc) == tuple(int(v) for v in d[f"c{i}_repack_meta"])
        np.testing.assert_array_equal(rw, d[f"c{i}_repack_words"])
        # serialized body = 24-byte header then the planes' little-endian words
        ser = d[f"c{i}_ser"]
        assert ser[:4].tobytes() == b"QGTC"
        np.testing.assert_array_equal(ser[24:].view("<u4").reshape(words.shape), words)


def test_single_bit_word_kats():
    # test_bitpack.py:45-56 / 80-90: a lone bit lands in bit 0 / bit 31
    a = np.zeros((1, 32), np.uint8)
    a[0, 0] = 1
    assert O.pack_words(a, O.COL)[0][0] == 0x00000001
    a[0, 0], a[0, 31] = 0, 1
    assert O.pack_words(a, O.COL)[0][0] == 0x80000000


def test_bmm_and_counters():
    d = load("gemm")
    for i in range(int(d["n_bmm"])):
        dense, xp = d[f"b{i}_dense"], d[f"b{i}_xplanes"]
        aw, pr, pc = O.pack_words(dense, O.COL, 8)
        xw, xpr, xpc = O.pack_stack(xp, O.ROW, 8)
        adims = (dense.shape[0], dense.shape[1], pr, pc)
        xdims = (xp.shape[1], xp.shape[2], xpr, xpc)
        flags = O.zero_tile_flags(aw, pr, pc)
        np.testing.assert_array_equal(flags, d[f"b{i}_flags"])
        for jump in (True, False):
            outs = O.bmm_planes(aw, adims, xw, xdims, jump=jump)
            np.testing.assert_array_equal(np.stack(outs), d[f"b{i}_out"])
        k = 0
        for jump in (True, False):
            for ct in (True, False):
                c = O.counters_bmm(flags, xp.shape[0], xpc // 8, jump=jump, cross_tile=ct)
                assert [c[f] for f in ("tile_mma_count", "tile_fetch_count", "tiles_skipped",
                                       "word_and_popcount_count", "tiles_total")] \
                    == list(d[f"b{i}_counters"][k])
                k += 1
        if f"b{i}_reduced" in d:
            np.testing.assert_array_equal(O.narrow_int32(O.shift_reduce(outs)), d[f"b{i}_reduced"])


def test_gemm_and_counters():
    d = load("gemm")
    for j in range(int(d["n_gemm"])):
        xp, wp = d[f"g{j}_xplanes"], d[f"g{j}_wplanes"]
        xw, xpr, xpc = O.pack_stack(xp, O.COL, 8)
        ww, wpr, wpc = O.pack_stack(wp, O.ROW, 8)
        got = O.gemm_planes(xw, (xp.shape[1], xp.shape[2], xpr, xpc), ww,
                            (wp.shape[1], wp.shape[2], wpr, wpc))
        np.testing.assert_array_equal(O.narrow_int32(got), d[f"g{j}_out"])
        flags = [O.zero_tile_flags(w, xpr, xpc) for w in xw]
        k = 0
        for jump in (True, False):
            for ct in (True, False):
                c = O.counters_gemm(flags, wp.shape[0], wpc // 8, jump=jump, cross_tile=ct)
                assert [c[f] for f in ("tile_mma_count", "tile_fetch_count", "tiles_skipped",
                                       "word_and_popcount_count", "tiles_total")] \
                    == list(d[f"g{j}_counters"][k])
                k += 1


def test_gemm_overflow_is_detected():
    # test_bitgemm.py:397-404: 255*255*33100 > 2**31-1 must not wrap
    k = 33100
    xw, xpr, xpc = O.pack_stack(np.ones((8, 1, k), np.uint8), O.COL, 8)
    ww, wpr, wpc = O.pack_stack(np.ones((8, k, 1), np.uint8), O.ROW, 8)
    total = O.gemm_planes(xw, (1, k, xpr, xpc), ww, (k, 1, wpr, wpc))
    assert int(total[0, 0]) == 255 * 255 * k
    assert O.narrow_int32(total) is None


def _grid_tuple(d, key):
    if key not in d:
        return None, None
    lo, hi, bits = d[key]
    return (lo, (hi - lo) / (1 << int(bits))), (lo, hi, int(bits))


def test_epilogue():
    d = load("epilogue")
    for i in range(int(d["n"])):
        p = f"e{i}_"
        lhs, _ = _grid_tuple(d, p + "lhs")
        rhs, _ = _grid_tuple(d, p + "rhs")
        real = O.dequantize(d[p + "acc"], lhs, rhs, d[p + "rows"], d[p + "cols"], int(d[p + "inner"]))
        bn = None
        if p + "bn" in d:
            mean, var, gamma, beta = d[p + "bn"]
            bn = (mean, var, gamma, beta, 1e-5)
        kind = str(d[p + "kind"])
        real = O.finish(real, d[p + "bias"] if p + "bias" in d else None, bn,
                        kind if kind != "batch-norm" else "none")
        _, outp = _grid_tuple(d, p + "outp")
        if outp is None:
            np.testing.assert_array_equal(real, d[p + "real"])
            continue
        codes = O.quantize_codes(real, *outp)
        np.testing.assert_array_equal(codes, d[p + "codes"])
        for orient, tag in ((O.ROW, "row"), (O.COL, "col")):
            words, pr, pc = O.pack_stack(O.planes_of(codes, outp[2]), orient, 8)
            assert (pr, pc) == tuple(int(v) for v in d[p + tag + "_dims"])
            np.testing.assert_array_equal(words, d[p + tag + "_words"])


@pytest.mark.parametrize("i", range(6))
def test_model_forward_matches_reference_logits(i):
    d = load("model")
    c = model_case(d, i)
    xg = c.x_params
    codes = O.quantize_codes(c.feats, xg.alpha_min, xg.alpha_max, xg.bits)
    # the batch's packed feature planes are the reference's row-wise packing of these codes
    fw, _, _ = O.pack_stack(O.planes_of(codes, xg.bits), O.ROW, 8)
    np.testing.assert_array_equal(fw, c.feat_words)
    np.testing.assert_array_equal(
        O.row_degrees(c.adj_words, c.adj_dims[2], c.adj_dims[3], c.adj_dims[0]), c.degrees)
    logits = O.model_forward(c.adj_words, c.adj_dims, codes, xg, c.layers)
    np.testing.assert_array_equal(logits, c.logits)
    dense = O.unpack_words(c.adj_words, O.COL, *c.adj_dims)
    np.testing.assert_array_equal(O.dense_int_forward(dense, codes, xg, c.layers), c.logits)
