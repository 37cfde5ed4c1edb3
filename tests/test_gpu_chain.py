"""Chained stage pairs (qg_chain): an aggregation whose requantized codes stay in shared
memory as the left operand of the following update GEMM, in one launch.  GCN chains
aggregate -> update inside a layer, GIN chains the aggregation of layer l with the
update of layer l + 1.  The chained forward must equal the two-launch forward (itself
checked against the reference oracle's logits elsewhere) bit for bit."""

import numpy as np
import pytest

from paper_2111_09547_b200 import bitgemm, engine, synth
from paper_2111_09547_b200.synth import GraphConfig

pytestmark = pytest.mark.gpu


def _forward(batches, model, chain):
    saved = engine.CHAIN
    engine.CHAIN = chain
    hook = []
    bitgemm.PROFILE_HOOK = hook
    try:
        outs = engine.model_forward_group(batches, model)
    finally:
        engine.CHAIN = saved
        bitgemm.PROFILE_HOOK = None
    return [o.cpu().numpy() for o in outs], len(hook)


# (model, in_dim, hidden, classes, layers, bits, wbits): stage widths below / above 128
# (two shared-memory K tiles), 256-wide accumulators, odd class counts, 1..8 bits
CASES = [
    ("gin", 128, 64, 39, 3, 4, 4),
    ("gin", 100, 256, 47, 3, 8, 8),
    ("gin", 40, 200, 7, 2, 2, 3),
    ("gin", 64, 32, 5, 4, 1, 1),
    ("gcn", 128, 128, 40, 2, 4, 4),
    ("gcn", 200, 64, 9, 3, 3, 2),
    ("gcn", 256, 16, 3, 2, 8, 8),
    ("gcn", 24, 256, 33, 2, 5, 6),
    ("gcn", 64, 16, 3, 2, 2, 2),        # C1-like: 16-column stage 2
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-{c[1]}-{c[2]}-{c[3]}x{c[4]}-b{c[5]}" for c in CASES])
def test_chained_forward_equals_two_launch_forward(case):
    """One CTA per row block runs both stages; the split two-launch path is the reference."""
    kind, in_dim, hidden, classes, layers, bits, wbits = case
    # 3 batches of 2 parts; 1237 nodes -> part sizes not multiples of 128 (ragged row blocks)
    cfg = GraphConfig("chain-test", kind, 1237, 9000, 6, 2, in_dim, hidden, classes, layers, bits, wbits)
    batches, feats, _ = synth.planted_batches(cfg, seed=3)
    model = synth.calibrated_model(cfg, batches[0], feats[0], seed=3)
    got, n_chained = _forward(batches, model, True)
    want, n_plain = _forward(batches, model, False)
    assert len(got) == len(want)
    for g, w in zip(got, want):
        np.testing.assert_array_equal(g, w)
    # GCN: at most one launch per layer instead of two; GIN: at most layers - 1 fewer launches
    # (_chain_ok keeps split stages with many row blocks on two launches)
    saved = layers if kind == "gcn" else layers - 1
    assert 0 <= n_plain - n_chained <= saved


def test_chained_forward_matches_oracle_small():
    """Direct oracle check of one chained GIN forward (small, CPU oracle in seconds)."""
    from oracle import qgtc_oracle as O
    cfg = GraphConfig("chain-oracle", "gin", 300, 1500, 2, 2, 48, 64, 6, 3, 3, 3)
    batches, feats, xp = synth.planted_batches(cfg, seed=5)
    model = synth.calibrated_model(cfg, batches[0], feats[0], seed=5)
    got, _ = _forward(batches, model, True)
    for b, f, g in zip(batches, feats, got):
        codes = O.quantize_codes(f, xp.alpha_min, xp.alpha_max, xp.bits)
        want = O.model_forward(b.adjacency.words, b.adjacency.dims(), codes, xp, model.layers)
        np.testing.assert_array_equal(g, want)


def test_chained_e2e_runner_equals_unchained_device_epoch():
    """The pipelined end-to-end runner (chained stages inside its per-chunk graphs) returns
    the logits of the two-launch device epoch, bit for bit."""
    import torch

    from paper_2111_09547_b200.runtime import EpochRunner, HostEpochRunner
    cfg = synth.with_bits(synth.CONFIGS["C3"], 4)
    batches, feats, _ = synth.planted_batches(cfg, seed=4, batch_ids=range(12))
    model = synth.calibrated_model(cfg, batches[0], feats[0], seed=4)
    saved = engine.CHAIN
    try:
        engine.CHAIN = False
        want = torch.cat([o.cpu() for o in EpochRunner(model, batches, rescan=False).capture().run()])
        engine.CHAIN = True
        host = HostEpochRunner(model, batches)
        assert host.chunks > 1
        for _ in range(2):
            out = host.run_host()
            host.stream.synchronize()
            assert torch.equal(out, want)
    finally:
        engine.CHAIN = saved


def test_op_counters_after_a_chained_forward():
    """op_counters() after a forward whose last op is a chained update (GCN) resolves to the
    same counters as after the two-launch forward (bitgemm.py:95-100 semantics)."""
    cfg = GraphConfig("chain-counters", "gcn", 700, 4000, 4, 2, 64, 32, 5, 2, 3, 3)
    batches, feats, _ = synth.planted_batches(cfg, seed=6)
    model = synth.calibrated_model(cfg, batches[0], feats[0], seed=6)
    _forward(batches, model, False)
    want = bitgemm.op_counters()
    _forward(batches, model, True)
    assert bitgemm.op_counters() == want


@pytest.mark.parametrize("kind", ["gcn", "gin"])
def test_chained_row_blocks_without_adjacency_blocks(kind):
    """A 128-row block with no non-zero adjacency block (isolated nodes, no self loops):
    the chained stage-1 tile has no MMA (zero accumulator) and its stage 2 still runs.
    Chained == two-launch == CPU oracle."""
    from oracle import qgtc_oracle as O
    from paper_2111_09547_b200 import bitpack, graph
    cfg = GraphConfig("chain-empty", kind, 600, 3000, 2, 2, 48, 64, 7, 3, 3, 3)
    batches, feats, xp = synth.planted_batches(cfg, seed=8)
    b = batches[0]
    a = b.adjacency
    dense = O.unpack_words(np.asarray(a.words), O.COL, a.logical_rows, a.logical_cols, a.padded_rows,
                           a.padded_cols)
    dense[128:256, :] = 0                                   # row block 1: no edges at all
    words, pr, pc = O.pack_words(dense, O.COL, 8)
    adj = bitpack.PackedBitMatrix(bitpack.COLUMN_WISE, a.logical_rows, a.logical_cols, pr, pc, words)
    nb = graph.SubgraphBatch(node_ids=b.node_ids, adjacency=adj, features=b.features, boundaries=b.boundaries,
                             x_params=b.x_params)
    model = synth.calibrated_model(cfg, nb, feats[0], seed=8)
    got, _ = _forward([nb], model, True)
    want, _ = _forward([nb], model, False)
    np.testing.assert_array_equal(got[0], want[0])
    codes = O.quantize_codes(feats[0], xp.alpha_min, xp.alpha_max, xp.bits)
    np.testing.assert_array_equal(got[0], O.model_forward(words, (a.logical_rows, a.logical_cols, pr, pc), codes,
                                                          xp, model.layers))
