"""GPU parity: the CUDA path vs the reference's golden vectors and the CPU oracle.

Every comparison is bit-exact (integers, packed words, requantized codes and
the fp64 logits: the epilogue evaluates the reference's fp64 expression
without contraction, so logits are compared with array_equal).
"""

import numpy as np
import pytest

import paper_2111_09547_b200 as bg
from golden_io import load, model_case
from oracle import qgtc_oracle as O

pytestmark = pytest.mark.gpu


def _qp(arr):
    return bg.QuantParams(float(arr[0]), float(arr[1]), int(arr[2]))


def test_quantize_matches_golden():
    d = load("quantize")
    for x, g, want in zip(d["kat_in"], d["kat_grid"], d["kat_out"]):
        assert bg.quantize_matrix([[x]], _qp(g)).values[0, 0] == want
    for i in range(int(d["n_matrix"])):
        qm = bg.quantize_matrix(d[f"m{i}_in"], _qp(d[f"m{i}_grid"]))
        np.testing.assert_array_equal(qm.values, d[f"m{i}_codes"])


def test_quantize_float32_source_equals_float64():
    rng = np.random.default_rng(3)
    m = rng.uniform(-1, 2, (300, 77)).astype(np.float32)
    import torch
    p = bg.QuantParams(-0.5, 1.5, 5)
    a = bg.quantize_matrix(torch.from_numpy(m).cuda(), p).values
    b = bg.quantize_matrix(m.astype(np.float64), p).values
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(a, O.quantize_codes(m, -0.5, 1.5, 5))


def test_nonfinite_reports_first_position():
    m = np.zeros((4, 5))
    m[2, 3] = np.nan
    m[3, 0] = np.inf
    with pytest.raises(bg.DataError, match=r"\(2, 3\)"):
        bg.quantize_matrix(m, bg.QuantParams(0.0, 1.0, 2))


def test_pack_repack_serialize_match_golden():
    d = load("pack")
    for i in range(int(d["n"])):
        planes = d[f"c{i}_planes"]
        o, pad, pr, pc = (int(v) for v in d[f"c{i}_meta"])
        orient = bg.COLUMN_WISE if o == 0 else bg.ROW_WISE
        st = bg.pack_planes(planes, orient, pad_to=pad)
        assert (st.padded_rows, st.padded_cols) == (pr, pc)
        np.testing.assert_array_equal(np.stack([p.words for p in st.planes]), d[f"c{i}_words"])
        np.testing.assert_array_equal(bg.to_planes(st), planes)
        assert bg.serialize(st) == d[f"c{i}_ser"].tobytes()
        assert bg.deserialize(d[f"c{i}_ser"].tobytes()) == st
        other = bg.ROW_WISE if orient == bg.COLUMN_WISE else bg.COLUMN_WISE
        rp = bg.repack(st, other)
        assert (rp.padded_rows, rp.padded_cols) == tuple(int(v) for v in d[f"c{i}_repack_meta"])
        np.testing.assert_array_equal(np.stack([p.words for p in rp.planes]), d[f"c{i}_repack_words"])


def test_single_bit_words_and_nonbinary():
    a = np.zeros((1, 32), np.uint8)
    a[0, 0] = 1
    assert bg.pack_colwise(a).words[0] == 0x00000001
    a[0, 0], a[0, 31] = 0, 1
    assert bg.pack_colwise(a).words[0] == 0x80000000
    b = np.zeros((3, 4), np.uint8)
    b[1, 2] = 2
    with pytest.raises(bg.DataError, match=r"\(1, 2\)"):
        bg.pack_colwise(b)


def test_bmm_outputs_counters_and_flags_match_golden():
    d = load("gemm")
    combos = [(True, bg.CROSS_TILE), (True, bg.CROSS_BIT), (False, bg.CROSS_TILE), (False, bg.CROSS_BIT)]
    for i in range(int(d["n_bmm"])):
        a = bg.pack_colwise(d[f"b{i}_dense"])
        xs = bg.pack_planes(d[f"b{i}_xplanes"], bg.ROW_WISE)
        np.testing.assert_array_equal(bg.scan_zero_tiles(a).flags, d[f"b{i}_flags"])
        for k, (jump, reuse) in enumerate(combos):
            outs = bg.bmm_1bit_by_nbit(a, xs, jump=jump, reuse=reuse)
            np.testing.assert_array_equal(np.stack(outs), d[f"b{i}_out"])
            c = bg.op_counters()
            assert [c.tile_mma_count, c.tile_fetch_count, c.tiles_skipped, c.word_and_popcount_count,
                    c.tiles_total] == list(d[f"b{i}_counters"][k])
        if f"b{i}_reduced" in d:
            np.testing.assert_array_equal(bg.reduce_bitplanes(outs), d[f"b{i}_reduced"])


def test_gemm_outputs_and_counters_match_golden():
    d = load("gemm")
    combos = [(True, bg.CROSS_TILE), (True, bg.CROSS_BIT), (False, bg.CROSS_TILE), (False, bg.CROSS_BIT)]
    for j in range(int(d["n_gemm"])):
        xs = bg.pack_planes(d[f"g{j}_xplanes"], bg.COLUMN_WISE)
        ws = bg.pack_planes(d[f"g{j}_wplanes"], bg.ROW_WISE)
        for k, (jump, reuse) in enumerate(combos):
            acc = bg.gemm_sbit_by_tbit(xs, ws, "int32", jump=jump, reuse=reuse)
            np.testing.assert_array_equal(acc, d[f"g{j}_out"])
            c = bg.op_counters()
            assert [c.tile_mma_count, c.tile_fetch_count, c.tiles_skipped, c.word_and_popcount_count,
                    c.tiles_total] == list(d[f"g{j}_counters"][k])


def test_gemm_overflow_raises():
    k = 33100  # 255*255*k > 2**31 - 1 (reference test_bitgemm.py:397-404)
    xs = bg.pack_planes(np.ones((8, 1, k), np.uint8), bg.COLUMN_WISE)
    ws = bg.pack_planes(np.ones((8, k, 1), np.uint8), bg.ROW_WISE)
    with pytest.raises(bg.ReductionOverflowError):
        bg.gemm_sbit_by_tbit(xs, ws, "int32")
    accs = [np.full((2, 2), 2 ** 28, dtype=np.int64) for _ in range(8)]
    with pytest.raises(bg.ReductionOverflowError):
        bg.reduce_bitplanes(accs)


def _epi_from_golden(d, p):
    def grid(k):
        return _qp(d[p + k]) if p + k in d else None
    bn = None
    if p + "bn" in d:
        mean, var, gamma, beta = d[p + "bn"]
        bn = bg.BatchNormParams(mean=mean, var=var, gamma=gamma, beta=beta)
    return bg.EpilogueSpec(kind=str(d[p + "kind"]), lhs_params=grid("lhs"), rhs_params=grid("rhs"),
                           lhs_row_sums=d[p + "rows"], rhs_col_sums=d[p + "cols"], inner_dim=int(d[p + "inner"]),
                           bias=d[p + "bias"] if p + "bias" in d else None, bn=bn, out_params=grid("outp"))


def test_epilogue_matches_golden():
    d = load("epilogue")
    for i in range(int(d["n"])):
        p = f"e{i}_"
        epi = _epi_from_golden(d, p)
        if epi.out_params is None:
            np.testing.assert_array_equal(bg.apply_epilogue(d[p + "acc"], epi), d[p + "real"])
            continue
        for orient, tag in ((bg.ROW_WISE, "row"), (bg.COLUMN_WISE, "col")):
            st = bg.apply_epilogue(d[p + "acc"], epi, out_orientation=orient)
            assert (st.padded_rows, st.padded_cols) == tuple(int(v) for v in d[p + tag + "_dims"])
            np.testing.assert_array_equal(np.stack([q.words for q in st.planes]), d[p + tag + "_words"])


def test_fused_equals_unfused_epilogue():
    rng = np.random.default_rng(22)
    for (m, k, n, s, t) in [(20, 150, 10, 3, 2), (300, 257, 64, 4, 4), (130, 128, 200, 8, 8)]:
        xs = bg.pack_planes((rng.uniform(0, 1, (s, m, k)) < 0.5).astype(np.uint8), bg.COLUMN_WISE)
        ws = bg.pack_planes((rng.uniform(0, 1, (t, k, n)) < 0.5).astype(np.uint8), bg.ROW_WISE)
        bn = bg.BatchNormParams(mean=rng.uniform(-1, 1, n), var=rng.uniform(0.5, 2, n),
                                gamma=rng.uniform(0.5, 1.5, n), beta=rng.uniform(-1, 1, n))
        epi = bg.EpilogueSpec(kind="relu", lhs_params=bg.QuantParams(-0.3, 1.0, s),
                              rhs_params=bg.QuantParams(-0.5, 0.5, t), lhs_row_sums=rng.integers(0, 50, m),
                              rhs_col_sums=rng.integers(0, 50, n), inner_dim=k, bias=rng.uniform(-1, 1, n),
                              bn=bn, out_params=bg.QuantParams(-2.0, 40.0, 5))
        for orient in (bg.ROW_WISE, bg.COLUMN_WISE):
            fused = bg.gemm_sbit_by_tbit(xs, ws, "bitplanes", epi, out_orientation=orient)
            acc = bg.gemm_sbit_by_tbit(xs, ws, "int32")
            assert fused == bg.apply_epilogue(acc, epi, out_orientation=orient)


def _model_from_case(c):
    layers = []
    for ly in c.layers:
        bn = None
        if ly.bn is not None:
            bn = bg.BatchNormParams(mean=ly.bn.mean, var=ly.bn.var, gamma=ly.bn.gamma, beta=ly.bn.beta,
                                    eps=ly.bn.eps)
        g = ly.weight_params
        layers.append(bg.LayerConfig(
            in_dim=ly.in_dim, out_dim=ly.out_dim, weight=ly.weight,
            weight_params=bg.QuantParams(g.alpha_min, g.alpha_max, g.bits), bias=ly.bias,
            activation=ly.activation, bn=bn, order=ly.order, output_mode=ly.output_mode,
            mid_params=bg.QuantParams(ly.mid_params.alpha_min, ly.mid_params.alpha_max, ly.mid_params.bits),
            out_params=None if ly.out_params is None else bg.QuantParams(
                ly.out_params.alpha_min, ly.out_params.alpha_max, ly.out_params.bits)))
    kind = "cluster-gcn" if c.kind == "gcn" else "batched-gin"
    return bg.ModelConfig(layers=layers, kind=kind, feature_bits=c.x_params.bits,
                          weight_bits=layers[0].weight_params.bits)


def _batch_from_case(c):
    n = c.adj_dims[0]
    adj = bg.PackedBitMatrix(bg.COLUMN_WISE, *c.adj_dims, c.adj_words)
    fr, fc = c.feats.shape
    planes = [bg.PackedBitMatrix(bg.ROW_WISE, fr, fc, bg.pad128(fr), bg.pad8(fc), w) for w in c.feat_words]
    feats = bg.BitPlaneStack(bits=len(planes), planes=planes)
    xg = c.x_params
    return bg.SubgraphBatch(node_ids=c.node_ids, adjacency=adj, features=feats, boundaries=c.boundaries,
                            x_params=bg.QuantParams(xg.alpha_min, xg.alpha_max, xg.bits)), n


@pytest.mark.parametrize("i", range(6))
def test_model_forward_matches_reference_logits(i):
    c = model_case(load("model"), i)
    batch, _ = _batch_from_case(c)
    model = _model_from_case(c)
    np.testing.assert_array_equal(batch.degrees(), c.degrees)
    tally = bg.KernelTally()
    logits = bg.model_forward(batch, model, tally=tally)
    np.testing.assert_array_equal(logits, c.logits)
    got = [[t.tile_mma_count, t.tile_fetch_count, t.tiles_skipped, t.word_and_popcount_count, t.tiles_total]
           for t in (tally.total, tally.aggregation)]
    np.testing.assert_array_equal(np.array(got), c.tally)
    # ablations are output-invariant (cli.py:224-228): dense schedule + CUDA-core bit-serial path
    for jump, reuse in ((False, bg.CROSS_TILE), (True, bg.CROSS_BIT), (False, bg.CROSS_BIT)):
        np.testing.assert_array_equal(bg.model_forward(batch, model, jump=jump, reuse=reuse), c.logits)


@pytest.mark.parametrize("i", range(6))
def test_compound_buffer_roundtrip_matches_golden(i):
    c = model_case(load("model"), i)
    batch, _ = _batch_from_case(c)
    buf = bg.pack_batch(batch)
    assert buf.data == c.compound
    back = bg.unpack_batch(buf)
    assert back == batch
    np.testing.assert_array_equal(bg.model_forward(back, _model_from_case(c)), c.logits)


@pytest.mark.parametrize("i", range(6))
def test_tile_sparse_wire_format_roundtrip(i):
    """QGT3 (schedule + non-zero 128x128 blocks only): the rebuilt dense words equal the
    original adjacency, and the end-to-end runner (one graph: H2D -> epoch -> D2H)
    reproduces the reference logits bit for bit."""
    import torch

    from paper_2111_09547_b200 import graph
    from paper_2111_09547_b200.runtime import HostEpochRunner
    c = model_case(load("model"), i)
    batch, _ = _batch_from_case(c)
    img = graph.pack_batch_v3(batch)
    dev = torch.from_numpy(np.frombuffer(img, dtype=np.uint8).copy()).cuda()
    back = graph.batch_from_v3(img, dev, 0)
    np.testing.assert_array_equal(back.adjacency.words, batch.adjacency.words)
    assert back.features == batch.features
    np.testing.assert_array_equal(back.degrees(), batch.degrees())
    model = _model_from_case(c)
    np.testing.assert_array_equal(bg.model_forward(back, model), c.logits)
    host = HostEpochRunner(model, [batch])
    assert host.h2d_bytes == len(img)
    for _ in range(2):
        out = host.run_host()
        host.stream.synchronize()
        np.testing.assert_array_equal(out.numpy(), c.logits)


def test_bindings_match_golden():
    from paper_2111_09547_b200 import bindings as bb
    d = load("bindings")
    for i in range(int(d["n"])):
        sa, sb = (int(v) for v in d[f"h{i}_bits"])
        ha, hb = bb.to_bit(d[f"h{i}_a"], sa), bb.to_bit(d[f"h{i}_b"], sb)
        np.testing.assert_array_equal(bb.to_val(ha), d[f"h{i}_a_codes"])
        np.testing.assert_array_equal(np.stack([p.words for p in ha._stack(bg.COLUMN_WISE).planes]),
                                      d[f"h{i}_a_words"])
        np.testing.assert_array_equal(bb.bitMM2Int(ha, hb), d[f"h{i}_int"])
        hc = bb.bitMM2Bit(ha, hb, 4)
        np.testing.assert_array_equal(bb.to_val(hc), d[f"h{i}_bit4_codes"])
        np.testing.assert_array_equal([hc.params.alpha_min, hc.params.alpha_max, hc.params.bits],
                                      d[f"h{i}_bit4_grid"])
    ha.release()
    with pytest.raises(ValueError, match="released"):
        bb.to_val(ha)


@pytest.mark.parametrize("variant", ["no_chain", "default"])
@pytest.mark.parametrize("i", [0, 3, 5])
def test_engine_variants_match_golden(variant, i):
    """Chained (default) and two-launch (unchained) stage pairs stay bit-exact against the
    reference logits."""
    from paper_2111_09547_b200 import engine
    c = model_case(load("model"), i)
    batch, _ = _batch_from_case(c)
    model = _model_from_case(c)
    saved = engine.CHAIN
    try:
        engine.CHAIN = variant != "no_chain"
        np.testing.assert_array_equal(bg.model_forward(batch, model), c.logits)
    finally:
        engine.CHAIN = saved


def test_pipelined_e2e_runner_equals_single_graph():
    """The chunked e2e runner (H2D / compute / D2H of batch chunks overlapped on two copy
    engines) returns the same fp64 logits as the single-transfer runner, bit for bit."""
    import torch

    from paper_2111_09547_b200 import synth
    from paper_2111_09547_b200.runtime import HostEpochRunner
    cfg = synth.with_bits(synth.CONFIGS["C3"], 4)
    batches, feats, _ = synth.planted_batches(cfg, seed=2, batch_ids=range(10))
    model = synth.calibrated_model(cfg, batches[0], feats[0], seed=2)
    one = HostEpochRunner(model, batches, chunks=1)
    piped = HostEpochRunner(model, batches, chunks=3)
    assert piped.chunks == 3
    a = one.run_host()
    one.stream.synchronize()
    for _ in range(2):
        b = piped.run_host()
        piped.stream.synchronize()
        assert torch.equal(a, b)
    dev = torch.cat([o.cpu() for o in bg.engine.model_forward_group(batches, model)])
    assert torch.equal(a, dev)
