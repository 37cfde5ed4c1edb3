"""Generate golden vectors by running the REAL reference (``bitgnn``) here.

The reference is pure Python/numpy and cannot travel to the GPU box, so its
outputs on seeded inputs are frozen into ``tests/golden/*.npz`` and committed.
Run from the repo root (needs /root/reference, i.e. only in the build
container):

    python tests/golden/make_golden.py

Every case stores its inputs and the reference outputs; tests read them back
and compare the oracle (CPU) and the CUDA path (GPU) against them.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
REF_BIND = "/root/reference/pkg/bindings/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _load_reference():
    sys.path.insert(0, REF_BIND)
    sys.path.insert(0, REF)
    import bitgnn  # noqa: E402  (the reference package)
    import bitgnn_bindings  # noqa: E402
    return bitgnn, bitgnn_bindings


def quantize_cases(bg, rng):
    d = {}
    kats = [(5.7, 0.0, 8.0, 3), (0.49, -1.0, 1.0, 2), (1.0, -1.0, 1.0, 3), (-3.0, 0.0, 1.0, 4),
            (0.0, 0.0, 1.0, 1), (0.999999, 0.0, 1.0, 8)]
    d["kat_in"] = np.array([k[0] for k in kats])
    d["kat_grid"] = np.array([[k[1], k[2], k[3]] for k in kats])
    d["kat_out"] = np.array([bg.quantize_scalar(k[0], bg.QuantParams(k[1], k[2], k[3])) for k in kats])
    i = 0
    for bits in (1, 2, 3, 4, 5, 8):
        for (lo, hi) in ((0.0, 1.0), (-0.5, 0.5), (-1.3, 2.7)):
            r, c = int(rng.integers(1, 70)), int(rng.integers(1, 300))
            m = rng.uniform(lo - 0.2, hi + 0.2, (r, c))
            if i % 3 == 0:
                m = m.astype(np.float32).astype(np.float64)
            qm = bg.quantize_matrix(m, bg.QuantParams(lo, hi, bits))
            d[f"m{i}_in"] = m
            d[f"m{i}_grid"] = np.array([lo, hi, bits], dtype=np.float64)
            d[f"m{i}_codes"] = qm.values
            i += 1
    d["n_matrix"] = np.array(i)
    return d


def pack_cases(bg, rng):
    d = {}
    i = 0
    shapes = [(1, 1), (10, 200), (200, 64), (7, 129), (130, 33), (64, 256), (3, 300), (257, 5)]
    for (r, c) in shapes:
        for orient in (bg.COLUMN_WISE, bg.ROW_WISE):
            for pad in (8, 128):
                bits = int(rng.integers(1, 5))
                planes = (rng.uniform(0, 1, (bits, r, c)) < 0.4).astype(np.uint8)
                st = bg.pack_planes(planes, orient, pad_to=pad)
                d[f"c{i}_planes"] = planes
                d[f"c{i}_meta"] = np.array([0 if orient == bg.COLUMN_WISE else 1, pad,
                                            st.padded_rows, st.padded_cols])
                d[f"c{i}_words"] = np.stack([p.words for p in st.planes])
                d[f"c{i}_ser"] = np.frombuffer(bg.serialize(st), dtype=np.uint8)
                rp = bg.repack(st, bg.ROW_WISE if orient == bg.COLUMN_WISE else bg.COLUMN_WISE)
                d[f"c{i}_repack_words"] = np.stack([p.words for p in rp.planes])
                d[f"c{i}_repack_meta"] = np.array([rp.padded_rows, rp.padded_cols])
                i += 1
    d["n"] = np.array(i)
    return d


def _block_diag(rng, n, parts, density):
    dense = np.zeros((n, n), dtype=np.uint8)
    bounds = np.linspace(0, n, parts + 1).astype(int)
    for b in range(parts):
        lo, hi = bounds[b], bounds[b + 1]
        dense[lo:hi, lo:hi] = rng.uniform(0, 1, (hi - lo, hi - lo)) < density
    np.fill_diagonal(dense, 1)
    return dense


def gemm_cases(bg, rng):
    d = {}
    i = 0
    # bmm: adjacency x s-bit stack, all jump/reuse combinations recorded
    bmm_shapes = [(20, 300, 13, 3, "rand", 0.3), (64, 256, 32, 4, "rand", 0.3),
                  (100, 400, 20, 3, "rand", 0.05), (300, 300, 16, 2, "bd", 0.2),
                  (24, 300, 16, 3, "zero", 0.0), (80, 600, 8, 5, "rand", 0.01),
                  (520, 520, 64, 8, "bd", 0.1), (9, 140, 7, 1, "rand", 0.5)]
    for (m, k, n, s, kind, dens) in bmm_shapes:
        if kind == "bd":
            dense = _block_diag(rng, m, 4, dens)[:m, :k]
        elif kind == "zero":
            dense = np.zeros((m, k), dtype=np.uint8)
        else:
            dense = (rng.uniform(0, 1, (m, k)) < dens).astype(np.uint8)
        a = bg.pack_colwise(dense)
        xp = (rng.uniform(0, 1, (s, k, n)) < 0.5).astype(np.uint8)
        xs = bg.pack_planes(xp, bg.ROW_WISE)
        d[f"b{i}_dense"] = dense
        d[f"b{i}_xplanes"] = xp
        outs = bg.bmm_1bit_by_nbit(a, xs)
        d[f"b{i}_out"] = np.stack(outs)
        d[f"b{i}_flags"] = bg.scan_zero_tiles(a).flags
        cnt = []
        for jump in (True, False):
            for reuse in (bg.CROSS_TILE, bg.CROSS_BIT):
                bg.bmm_1bit_by_nbit(a, xs, jump=jump, reuse=reuse)
                c = bg.op_counters()
                cnt.append([c.tile_mma_count, c.tile_fetch_count, c.tiles_skipped,
                            c.word_and_popcount_count, c.tiles_total])
        d[f"b{i}_counters"] = np.array(cnt, dtype=np.int64)
        red = bg.reduce_bitplanes(outs) if s <= 8 else None
        d[f"b{i}_reduced"] = red
        i += 1
    d["n_bmm"] = np.array(i)
    j = 0
    gemm_shapes = [(32, 128, 16, 3, 2, 0.5), (1, 1, 1, 3, 2, 1.0), (50, 260, 12, 4, 3, 0.05),
                   (16, 140, 10, 1, 1, 0.5), (100, 157, 99, 8, 8, 0.5), (40, 200, 24, 2, 5, 0.5),
                   (130, 64, 200, 4, 4, 0.5), (7, 300, 129, 5, 3, 0.5)]
    for (m, k, n, s, t, dens) in gemm_shapes:
        xp = (rng.uniform(0, 1, (s, m, k)) < dens).astype(np.uint8)
        wp = (rng.uniform(0, 1, (t, k, n)) < 0.5).astype(np.uint8)
        xs = bg.pack_planes(xp, bg.COLUMN_WISE)
        ws = bg.pack_planes(wp, bg.ROW_WISE)
        d[f"g{j}_xplanes"] = xp
        d[f"g{j}_wplanes"] = wp
        d[f"g{j}_out"] = bg.gemm_sbit_by_tbit(xs, ws, "int32")
        cnt = []
        for jump in (True, False):
            for reuse in (bg.CROSS_TILE, bg.CROSS_BIT):
                bg.gemm_sbit_by_tbit(xs, ws, "int32", jump=jump, reuse=reuse)
                c = bg.op_counters()
                cnt.append([c.tile_mma_count, c.tile_fetch_count, c.tiles_skipped,
                            c.word_and_popcount_count, c.tiles_total])
        d[f"g{j}_counters"] = np.array(cnt, dtype=np.int64)
        j += 1
    d["n_gemm"] = np.array(j)
    return d


def epilogue_cases(bg, rng):
    d = {}
    i = 0
    QP = bg.QuantParams
    specs = []
    # (kind, lhs, rhs, bias, bn, out, acc_hi)
    specs.append(("relu", QP(-1.0, 1.0, 4), QP(-0.5, 0.5, 3), True, True, QP(-3.0, 3.0, 4), 40))
    specs.append(("none", None, QP(0.0, 1.0, 2), False, False, None, 10))
    specs.append(("tanh", None, QP(0.0, 1.0, 2), False, False, None, 10))
    specs.append(("none", None, QP(-0.7, 1.9, 5), False, False, QP(-2.0, 40.0, 6), 200))
    specs.append(("relu", QP(0.0, 1.0, 3), QP(0.0, 1.0, 2), False, False, QP(0.0, 40.0, 5), 60))
    specs.append(("batch-norm", QP(-0.3, 0.9, 8), QP(-0.5, 0.5, 8), True, True, None, 100000))
    specs.append(("tanh", QP(-0.3, 0.9, 4), QP(-0.5, 0.5, 4), True, True, QP(-1.0, 1.0, 7), 3000))
    for (kind, lhs, rhs, has_bias, has_bn, outp, hi) in specs:
        m, n = int(rng.integers(3, 40)), int(rng.integers(2, 40))
        acc = rng.integers(-hi // 4, hi, (m, n)).astype(np.int32)
        rows = rng.integers(0, 60, m)
        cols = rng.integers(0, 30, n)
        inner = int(rng.integers(1, 50))
        bias = rng.uniform(-0.5, 0.5, n) if has_bias else None
        bn = None
        if has_bn or kind == "batch-norm":
            bn = bg.BatchNormParams(mean=rng.uniform(-1, 1, n), var=rng.uniform(0.5, 2, n),
                                    gamma=rng.uniform(0.5, 1.5, n), beta=rng.uniform(-1, 1, n))
        epi = bg.EpilogueSpec(kind=kind, lhs_params=lhs, rhs_params=rhs, lhs_row_sums=rows,
                              rhs_col_sums=cols, inner_dim=inner, bias=bias, bn=bn,
                              out_params=outp)
        d[f"e{i}_acc"] = acc
        d[f"e{i}_rows"] = rows
        d[f"e{i}_cols"] = cols
        d[f"e{i}_inner"] = np.array(inner)
        d[f"e{i}_kind"] = np.array(kind)
        for nm, p in (("lhs", lhs), ("rhs", rhs), ("outp", outp)):
            if p is not None:
                d[f"e{i}_{nm}"] = np.array([p.alpha_min, p.alpha_max, p.bits])
        if bias is not None:
            d[f"e{i}_bias"] = bias
        if bn is not None:
            d[f"e{i}_bn"] = np.stack([bn.mean, bn.var, bn.gamma, bn.beta])
        if outp is None:
            d[f"e{i}_real"] = bg.apply_epilogue(acc, epi)
        else:
            for orient, tag in ((bg.ROW_WISE, "row"), (bg.COLUMN_WISE, "col")):
                st = bg.apply_epilogue(acc, epi, out_orientation=orient)
                d[f"e{i}_{tag}_words"] = np.stack([p.words for p in st.planes])
                d[f"e{i}_{tag}_dims"] = np.array([st.padded_rows, st.padded_cols])
            d[f"e{i}_codes"] = bg.to_val(bg.to_planes(st))
        i += 1
    d["n"] = np.array(i)
    return d


def _planted_graph(rng, n, parts, edges_per_node, dim):
    part_of = np.repeat(np.arange(parts), -(-n // parts))[:n]
    src = rng.integers(0, n, edges_per_node * n)
    # 80% intra-part edges: pick the destination inside the source's part
    dst = rng.integers(0, n, len(src))
    intra = rng.uniform(0, 1, len(src)) < 0.8
    size = -(-n // parts)
    dst[intra] = np.minimum(part_of[src[intra]] * size + rng.integers(0, size, intra.sum()), n - 1)
    edges = np.stack([np.concatenate([src, dst]), np.concatenate([dst, src])], axis=1)
    feats = rng.uniform(0.0, 1.0, (n, dim))
    return edges, part_of, feats


def model_cases(bg, rng):
    d = {}
    cfgs = [
        # kind, n, parts, batch parts, dim, hidden, classes, layers, bits_x, bits_w, bn, act_last
        ("gcn", 60, 3, (0, 1, 2), 10, 16, 5, 2, 2, 2, False),
        ("gin", 48, 3, (0, 1, 2), 10, 64, 4, 3, 4, 4, False),
        ("gcn", 300, 6, (1, 3, 4), 32, 16, 10, 3, 4, 4, True),
        ("gin", 280, 4, (0, 2, 3), 24, 64, 7, 3, 8, 8, True),
        ("gin", 200, 2, (0, 1), 128, 64, 39, 3, 1, 1, False),
        ("gcn", 180, 3, (2, 0), 40, 128, 9, 2, 3, 5, False),
    ]
    for i, (kind, n, parts, bparts, dim, hid, cls, nl, bx, bw, use_bn) in enumerate(cfgs):
        edges, part_of, feats = _planted_graph(rng, n, parts, 4, dim)
        g = bg.Graph(num_nodes=n, edges=edges, features=feats)
        assign = bg.PartitionAssignment(num_parts=parts, part_of=part_of)
        xp = bg.QuantParams(0.0, 1.0, bx)
        batch = bg.build_batch(g, assign, list(bparts), xp)
        builder = bg.gcn_model if kind == "gcn" else bg.gin_model
        model = builder(dim, cls, hidden_dim=hid, num_layers=nl, feature_bits=bx,
                        weight_bits=bw, seed=i)
        if use_bn:
            for ly in model.layers:
                ly.bn = bg.BatchNormParams(mean=rng.uniform(-0.2, 0.2, ly.out_dim),
                                           var=rng.uniform(0.5, 2.0, ly.out_dim),
                                           gamma=rng.uniform(0.5, 1.5, ly.out_dim),
                                           beta=rng.uniform(-0.1, 0.1, ly.out_dim))
        bfeats = feats[batch.node_ids]
        bg.calibrate_model(model, batch, bfeats)
        tally = bg.KernelTally()
        logits = bg.model_forward(batch, model, tally=tally)
        p = f"m{i}_"
        d[p + "kind"] = np.array(kind)
        d[p + "adj_words"] = batch.adjacency.words
        d[p + "adj_dims"] = np.array([batch.adjacency.logical_rows, batch.adjacency.logical_cols,
                                      batch.adjacency.padded_rows, batch.adjacency.padded_cols])
        d[p + "node_ids"] = batch.node_ids
        d[p + "boundaries"] = batch.boundaries
        d[p + "feats"] = bfeats
        d[p + "feat_words"] = np.stack([q.words for q in batch.features.planes])
        d[p + "x_grid"] = np.array([xp.alpha_min, xp.alpha_max, xp.bits])
        d[p + "n_layers"] = np.array(len(model.layers))
        for li, ly in enumerate(model.layers):
            q = f"{p}L{li}_"
            d[q + "w"] = ly.weight
            d[q + "b"] = ly.bias
            d[q + "wgrid"] = np.array([ly.weight_params.alpha_min, ly.weight_params.alpha_max,
                                       ly.weight_params.bits])
            d[q + "mid"] = np.array([ly.mid_params.alpha_min, ly.mid_params.alpha_max,
                                     ly.mid_params.bits])
            if ly.out_params is not None:
                d[q + "out"] = np.array([ly.out_params.alpha_min, ly.out_params.alpha_max,
                                         ly.out_params.bits])
            d[q + "meta"] = np.array([ly.in_dim, ly.out_dim,
                                      0 if ly.order == "aggregate-then-update" else 1,
                                      {"none": 0, "relu": 1, "tanh": 2}[ly.activation],
                                      0 if ly.output_mode == "bitplanes" else 1])
            if ly.bn is not None:
                d[q + "bn"] = np.stack([ly.bn.mean, ly.bn.var, ly.bn.gamma, ly.bn.beta])
                d[q + "bn_eps"] = np.array(ly.bn.eps)
        d[p + "logits"] = logits
        d[p + "tally"] = np.array([[c.tile_mma_count, c.tile_fetch_count, c.tiles_skipped,
                                    c.word_and_popcount_count, c.tiles_total]
                                   for c in (tally.total, tally.aggregation)], dtype=np.int64)
        d[p + "compound"] = np.frombuffer(bg.pack_batch(batch).data, dtype=np.uint8)
        d[p + "degrees"] = batch.degrees()
    d["n"] = np.array(len(cfgs))
    return d


def binding_cases(bg, bb, rng):
    d = {}
    for i in range(6):
        m, k, n = (int(v) for v in rng.integers(1, 90, 3))
        sa, sb = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        a = rng.uniform(-1, 1, (m, k))
        b = rng.uniform(0, 3, (k, n))
        ha, hb = bb.to_bit(a, sa), bb.to_bit(b, sb)
        d[f"h{i}_a"], d[f"h{i}_b"] = a, b
        d[f"h{i}_bits"] = np.array([sa, sb])
        d[f"h{i}_a_codes"] = bb.to_val(ha)
        d[f"h{i}_a_words"] = np.stack([p.words for p in ha._stack(bg.COLUMN_WISE).planes])
        d[f"h{i}_int"] = bb.bitMM2Int(ha, hb)
        hc = bb.bitMM2Bit(ha, hb, 4)
        d[f"h{i}_bit4_codes"] = bb.to_val(hc)
        d[f"h{i}_bit4_grid"] = np.array([hc.params.alpha_min, hc.params.alpha_max, hc.params.bits])
    d["n"] = np.array(6)
    return d


def partition_cases(bg, rng):
    """Reference partition() (graph.py:190-229) + edge_cut on random and planted graphs."""
    d = {}
    cases = []
    for _ in range(10):
        n = int(rng.integers(8, 300))
        cases.append((n, rng.integers(0, n, (int(rng.integers(0, 4 * n)), 2))))
    edges, _, _ = _planted_graph(rng, 600, 6, 4, 1)
    cases.append((600, edges))
    cases.append((5, np.zeros((0, 2), dtype=np.int64)))               # edgeless: seeds only
    for i, (n, e) in enumerate(cases):
        g = bg.Graph(n, e)
        d[f"g{i}_n"] = np.array(n)
        d[f"g{i}_edges"] = g.edges
        for parts in (1, 2, 5):
            for seed in (0, 7, 2 ** 33 + 5):
                if parts > n:
                    continue
                a = bg.partition(g, parts, seed=seed)
                d[f"g{i}_p{parts}_s{seed}"] = a.part_of
                d[f"g{i}_p{parts}_s{seed}_cut"] = np.array(a.edge_cut)
    d["n"] = np.array(len(cases))
    return d


def main():
    bg, bb = _load_reference()
    rng = np.random.default_rng(20261017)
    for name, fn in (("quantize", quantize_cases), ("pack", pack_cases), ("gemm", gemm_cases),
                     ("epilogue", epilogue_cases), ("model", model_cases)):
        d = fn(bg, rng)
        d = {k: v for k, v in d.items() if v is not None}
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
        print(name, len(d), "arrays")
    d = binding_cases(bg, bb, rng)
    np.savez_compressed(os.path.join(OUT, "bindings.npz"), **d)
    print("bindings", len(d), "arrays")
    # own generator: the fixtures above regenerate unchanged
    d = partition_cases(bg, np.random.default_rng(20261018))
    np.savez_compressed(os.path.join(OUT, "partition.npz"), **d)
    print("partition", len(d), "arrays")


if __name__ == "__main__":
    main()
