"""Kernel-level GPU checks beyond the golden fixtures: size-independent
properties at larger shapes (two independent device algorithms agree, exact
integer identities), the epilogue's fast division, and edge cases."""

import numpy as np
import pytest
import torch

import paper_2111_09547_b200 as bg
from oracle import qgtc_oracle as O
from paper_2111_09547_b200 import _native as N
from paper_2111_09547_b200 import bitgemm, synth

pytestmark = pytest.mark.gpu


def _div_check(a: np.ndarray, b: np.ndarray):
    y = 1.0 / b                                   # RN(1/b), IEEE on the host
    ta, tb, ty = (torch.from_numpy(np.ascontiguousarray(v)).cuda() for v in (a, b, y))
    out, ref = torch.empty_like(ta), torch.empty_like(ta)
    N.call("qg_test_div", N.ptr(ta), N.ptr(tb), N.ptr(ty), ta.numel(), N.ptr(out), N.ptr(ref), N.stream())
    out, ref = out.cpu().numpy(), ref.cpu().numpy()
    np.testing.assert_array_equal(ref, a / b)     # device IEEE == numpy IEEE
    same = (out.view(np.int64) == ref.view(np.int64)) | (np.isnan(out) & np.isnan(ref))
    assert same.all(), (a[~same][:5], b[~same][:5], out[~same][:5], ref[~same][:5])


def test_fast_division_is_correctly_rounded():
    rng = np.random.default_rng(0)
    n = 2_000_000
    # wide exponent range incl. the fallback regions
    a = rng.standard_normal(n) * np.exp2(rng.integers(-1060, 1020, n).astype(np.float64))
    b = np.abs(rng.standard_normal(n)) * np.exp2(rng.integers(-1060, 1020, n).astype(np.float64)) + 1e-300
    _div_check(a, b)
    # epilogue-like: quotients straddling integers (the floor() boundary) and grid scales
    b = rng.uniform(1e-6, 10.0, n)
    k = rng.integers(-10 ** 6, 10 ** 6, n).astype(np.float64)
    a = k * b
    a = np.where(rng.uniform(size=n) < 0.5, np.nextafter(a, np.inf), np.nextafter(a, -np.inf))
    _div_check(a, b)
    scales = np.array([(hi - lo) / (1 << bits) for lo, hi in [(-0.5, 0.5), (0.0, 1.0), (-3.1, 7.7)]
                       for bits in range(1, 9)])
    b = rng.choice(scales, n)
    a = rng.uniform(-50, 50, n)
    _div_check(a, b)
    specials = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 1.7e308, 1.0, 3.0])
    aa, bb = np.meshgrid(specials, np.array([1.0, 3.0, 0.1, 7e-310, 1e300]))
    _div_check(aa.ravel(), bb.ravel())


def _requant_check(x, amin, amax, bits):
    scale = (amax - amin) / (1 << bits)
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()
    out = torch.empty(t.numel(), dtype=torch.int32, device="cuda")
    ref = torch.empty_like(out)
    N.call("qg_test_requant", N.ptr(t), t.numel(), amin, scale, 1.0 / scale, bits, N.ptr(out), N.ptr(ref),
           N.stream())
    out, ref = out.cpu().numpy(), ref.cpu().numpy()
    np.testing.assert_array_equal(ref, O.quantize_codes(x, amin, amax, bits))   # device IEEE == numpy
    np.testing.assert_array_equal(out, ref)


def test_filtered_requant_is_bit_identical():
    rng = np.random.default_rng(11)
    n = 1_000_000
    for (amin, amax) in [(-0.5, 0.5), (0.0, 1.0), (-3.1, 7.7), (-1e-3, 2e-3), (0.0, 37.0), (-123.4, 567.8)]:
        for bits in (1, 2, 4, 7, 8):
            scale = (amax - amin) / (1 << bits)
            x = rng.uniform(amin - 0.3 * (amax - amin), amax + 0.3 * (amax - amin), n)
            _requant_check(x, amin, amax, bits)
            # far outside the grid (quotients beyond +-2^12 exercise the range clamps)
            far = np.concatenate([amin - rng.uniform(1, 10000, 4096) * scale, amin + rng.uniform(1, 10000, 4096) * scale])
            _requant_check(far, amin, amax, bits)
            # adversarial: exactly on and one ulp around every code boundary
            k = np.arange(-2, (1 << bits) + 3, dtype=np.float64)
            b = amin + k * scale
            edge = np.concatenate([b, np.nextafter(b, np.inf), np.nextafter(b, -np.inf),
                                   np.nextafter(np.nextafter(b, np.inf), np.inf),
                                   np.nextafter(np.nextafter(b, -np.inf), -np.inf)])
            _requant_check(edge, amin, amax, bits)
    specials = np.array([0.0, -0.0, np.nan, np.inf, -np.inf, 1e300, -1e300, 5e-324])
    _requant_check(specials, -0.5, 0.5, 4)


@pytest.mark.parametrize("bits", [1, 3, 8])
def test_tcgen05_matches_popc_at_scale(bits):
    # A 2048 x 4096 block-diagonal (zero-tile jumping active) x X (4096 x 200, `bits` planes)
    a = synth.bernoulli_adjacency(2048, 4096, 0.3, seed=bits, blocks=4)
    x, codes = synth.random_codes_stack(4096, 200, bits, bg.ROW_WISE, seed=bits)
    xs = bg.BitPlaneStack._wrap(bg.ROW_WISE, 4096, 200, x.padded_rows, x.padded_cols, x.dwords)
    tc = bitgemm.bmm_planes_device(a, xs, algo="tcgen05")
    pc = bitgemm.bmm_planes_device(a, xs, algo="popc")
    assert torch.equal(tc, pc)
    # reduced accumulator == A @ codes (exact in fp64 at these magnitudes)
    dense = torch.from_numpy(bg.unpack(a).astype(np.float64)).cuda()
    want = (dense @ codes.to(torch.float64)).to(torch.int64)
    red = torch.zeros_like(want)
    for p in range(bits):
        red += tc[p].to(torch.int64) << p
    assert torch.equal(red, want)


def test_reduced_gemm_matches_dense_product():
    for (m, k, n, s, t) in [(1000, 300, 129, 8, 8), (257, 1000, 64, 3, 5), (130, 128, 300, 2, 1)]:
        x, xc = synth.random_codes_stack(m, k, s, bg.COLUMN_WISE, seed=m)
        w, wc = synth.random_codes_stack(k, n, t, bg.ROW_WISE, seed=n)
        acc = bg.gemm_sbit_by_tbit(x, w, "int32")
        want = (xc.double() @ wc.double()).cpu().numpy().astype(np.int64)
        np.testing.assert_array_equal(acc, want)


def test_per_plane_cross_bit_and_cross_tile_agree():
    rng = np.random.default_rng(5)
    dense = (rng.uniform(0, 1, (300, 700)) < 0.1).astype(np.uint8)
    a = bg.pack_colwise(dense)
    xp = (rng.uniform(0, 1, (6, 700, 45)) < 0.5).astype(np.uint8)
    xs = bg.pack_planes(xp, bg.ROW_WISE)
    base = bg.bmm_1bit_by_nbit(a, xs, reuse=bg.CROSS_TILE)
    for jump in (True, False):
        outs = bg.bmm_1bit_by_nbit(a, xs, jump=jump, reuse=bg.CROSS_BIT)
        for p in range(6):
            np.testing.assert_array_equal(outs[p], base[p])
            np.testing.assert_array_equal(outs[p], dense.astype(np.int64) @ xp[p].astype(np.int64))


def test_repack_roundtrip_large():
    rng = np.random.default_rng(6)
    planes = (rng.uniform(0, 1, (5, 1000, 333)) < 0.5).astype(np.uint8)
    st = bg.pack_planes(planes, bg.ROW_WISE)
    col = bg.repack(st, bg.COLUMN_WISE)
    np.testing.assert_array_equal(bg.to_planes(col), planes)
    back = bg.repack(col, bg.ROW_WISE)
    assert back == st
    w, _, _ = O.pack_stack(planes, O.COL, 8)
    np.testing.assert_array_equal(np.stack([p.words for p in col.planes]), w)


def test_quantize_pack_large_matches_oracle():
    rng = np.random.default_rng(7)
    m = rng.uniform(-1, 2, (5000, 300))
    for bits in (1, 4, 8):
        p = bg.QuantParams(-0.5, 1.5, bits)
        for orient in (bg.ROW_WISE, bg.COLUMN_WISE):
            st = bg.pack_planes(bg.bit_decompose(bg.quantize_matrix(m, p)), orient)
            w, _, _ = O.pack_stack(O.planes_of(O.quantize_codes(m, -0.5, 1.5, bits), bits),
                                   O.COL if orient == bg.COLUMN_WISE else O.ROW, 8)
            np.testing.assert_array_equal(np.stack([q.words for q in st.planes]), w)


@pytest.mark.parametrize("bits,amin,amax", [(8, 0.0, 1.0), (4, -0.5, 1.5), (2, -3.0, 1.0), (8, -1e-3, 3e-3),
                                            (7, 100.0, 228.0)])
def test_bitqnt_fp32_screen_matches_oracle(bits, amin, amax):
    """The row-wise bit_qnt kernel's fp32 screen (fp32 sources) against the fp64
    reference quotient: random values, values exactly on and one float ulp around every
    code boundary (the exact path), out-of-range values; planes and row sums."""
    from paper_2111_09547_b200 import _native as N
    from paper_2111_09547_b200.quantize import quantize_pack_device
    rng = np.random.default_rng(bits)
    scale = (amax - amin) / (1 << bits)
    rows, cols = 3001, 100
    x = rng.uniform(amin - 0.2 * (amax - amin), amax + 0.2 * (amax - amin), (rows, cols)).astype(np.float32)
    k = np.arange(-1, (1 << bits) + 2, dtype=np.float64)
    edge = (amin + k * scale).astype(np.float32)
    edge = np.concatenate([edge, np.nextafter(edge, np.float32(np.inf)), np.nextafter(edge, np.float32(-np.inf))])
    flat = x.reshape(-1)
    flat[:len(edge)] = edge
    rng.shuffle(flat)
    x = flat.reshape(rows, cols)
    p = bg.QuantParams(amin, amax, bits)
    r = quantize_pack_device(x, p, N.ROW_WISE_ID, 8, row_sums=True)
    codes = O.quantize_codes(x.astype(np.float64), amin, amax, bits)
    w, _, _ = O.pack_stack(O.planes_of(codes, bits), O.ROW, 8)
    np.testing.assert_array_equal(r["planes"].cpu().numpy().view(np.uint32).reshape(w.shape), w)
    np.testing.assert_array_equal(r["row_sums"].cpu().numpy(), codes.astype(np.int64).sum(axis=1))


def test_empty_and_degenerate_shapes():
    a = bg.pack_colwise(np.zeros((0, 5), np.uint8))
    assert a.padded_rows == 0 and len(a.words) == 0
    x = bg.pack_planes(np.ones((2, 5, 3), np.uint8), bg.ROW_WISE)
    outs = bg.bmm_1bit_by_nbit(a, x)
    assert all(o.shape == (0, 3) for o in outs)
    one = bg.pack_colwise(np.ones((1, 1), np.uint8))
    y = bg.pack_planes(np.ones((8, 1, 1), np.uint8), bg.ROW_WISE)
    assert [int(o[0, 0]) for o in bg.bmm_1bit_by_nbit(one, y)] == [1] * 8


@pytest.mark.parametrize("side", ["left", "right"])
def test_grouped_entry_tiles_equal_per_batch_conversion(side):
    """qg_entry_tiles (one launch over ragged batches) == the per-batch planes->codes->tiles
    path, byte for byte including zero padding, and the row code sums match."""
    from paper_2111_09547_b200 import tiled
    rng = np.random.default_rng(11)
    stacks, codes = [], []
    for rows, cols, bits in ((1, 1, 3), (129, 100, 3), (300, 257, 3), (1000, 128, 3)):
        c = rng.integers(0, 1 << bits, (rows, cols), dtype=np.uint8)
        codes.append(c)
        stacks.append(bg.pack_planes(O.planes_of(c, bits), bg.ROW_WISE))
    keep = []
    got = tiled.entry_tiles(stacks, side, True, keep)
    assert got is not None
    for st, c, (tiles, pitch, rs) in zip(stacks, codes, got):
        want, wpitch = tiled.tiles_from_codes(torch.from_numpy(c).cuda(), c.shape[0], c.shape[1], c.shape[1], side)
        assert pitch == wpitch
        assert torch.equal(tiles, want)
        if side == "left":
            np.testing.assert_array_equal(rs.cpu().numpy(), c.astype(np.int64).sum(axis=1))


@pytest.mark.parametrize("bits", [1, 3, 8])
def test_bmm_reduced_equals_reduced_per_plane_bmm(bits):
    """tiled.bmm_reduced (C5 path) == reduce_bitplanes(bmm_1bit_by_nbit) of the reference
    API, with a block-diagonal A so zero-tile jumping skips whole row blocks."""
    from paper_2111_09547_b200 import tiled
    rng = np.random.default_rng(bits)
    m, k, n = 700, 900, 300
    dense = (rng.uniform(0, 1, (m, k)) < 0.05).astype(np.uint8)
    dense[:256, 600:] = 0
    dense[256:, :300] = 0
    x = rng.integers(0, 1 << bits, (k, n), dtype=np.uint8)
    a = bg.pack_colwise(dense)
    xs = bg.pack_planes(O.planes_of(x, bits), bg.ROW_WISE)
    got = tiled.bmm_reduced(a, xs).cpu().numpy()
    want = bg.reduce_bitplanes(bg.bmm_1bit_by_nbit(a, xs))
    np.testing.assert_array_equal(got, want)
    np.testing.assert_array_equal(got, dense.astype(np.int64) @ x.astype(np.int64))


@pytest.mark.parametrize("pair,m", [(True, 4000), (False, 4000), (True, 2900)])
def test_bmm_reduced_pair_path_large(pair, m):
    """The 2-SM (cta_group::2, TMA-signalled) pair path of bmm_reduced at a size that
    selects it: block-sparse A with empty row blocks (union schedule + zero blocks) and
    an odd number of row blocks; result == dense product, and == the single-CTA path.
    m = 4000: 32 row blocks = two full N-major groups of 8 pairs; m = 2900: 23 row blocks
    = 12 pairs, a short last group and a pair with one row block past the end."""
    from paper_2111_09547_b200 import tiled
    g = torch.Generator(device="cuda").manual_seed(3)
    k, n, bits = 2500, 4096, 5
    dense = (torch.rand((m, k), generator=g, device="cuda") < 0.02).to(torch.uint8)
    dense[:1000, 1200:] = 0
    dense[2600:3000] = 0                                  # empty row blocks (m = 4000)
    dense[2000:2300] = 0 if m < 4000 else dense[2000:2300]
    dense[3000:, :600] = 0
    codes = torch.randint(0, 1 << bits, (k, n), generator=g, device="cuda", dtype=torch.uint8)
    a = bg.pack_colwise(dense)
    tiles, pitch = tiled.tiles_from_codes(codes, k, n, n, "right")
    x = tiled.TiledCodeStack(bg.ROW_WISE, k, n, bits, tiles, "right", pitch)
    old = tiled.PAIR
    tiled.PAIR = pair
    try:
        got = tiled.bmm_reduced(a, x)
    finally:
        tiled.PAIR = old
    want = (dense.double() @ codes.double()).to(torch.int64)
    assert torch.equal(got.to(torch.int64), want)
