"""GPU batch construction vs the REAL reference's build_batch (graph.py:308-357).

* ``synth.planted_batches`` (edges -> packed words on the GPU, fused bit_qnt of
  the features) must produce the byte-identical QGTB compound buffer
  (``pack_batch``, graph.py:374-397) that the reference's ``build_batch`` +
  ``pack_batch`` produce from the same host edge list and features -- for the
  C1 batch and for a full-size C4 batch (13,061 nodes, 8 parts).
* ``graph.build_batch`` (GPU) on random graphs with random partitions, with and
  without self loops, must equal the reference's batch byte for byte.

Skipped when the reference is not staged (oracle/make_ref.py).
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def _ref():
    import ref_inputs
    R = ref_inputs.ref_module()
    if R is None:
        pytest.skip("oracle/_ref not staged")
    return R, ref_inputs


@pytest.mark.gpu
@pytest.mark.parametrize("name,b", [("C1", 0), ("C3", 187), ("C4", 0)])
def test_planted_batch_equals_reference_build_batch(name, b):
    import paper_2111_09547_b200 as bg
    from paper_2111_09547_b200 import synth
    from paper_2111_09547_b200 import synth_host as H
    R, ri = _ref()
    cfg = H.CONFIGS[name]
    ours, _, _ = synth.planted_batches(cfg, seed=0, batch_ids=[b])
    edges, bnd, x = H.host_batch(cfg, 0, b)
    ref = ri.ref_build(R, cfg, edges, bnd, x)
    want = R.pack_batch(ref).data
    # node ids: the reference numbers the batch's own graph from 0, ours keeps global ids
    ours[0].node_ids = np.arange(ours[0].total_nodes)
    got = bg.pack_batch(ours[0]).data
    assert len(got) == len(want)
    assert got == want


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6))
def test_build_batch_random_graphs(seed):
    import paper_2111_09547_b200 as bg
    R, _ = _ref()
    rng = np.random.default_rng(seed)
    n = int(rng.integers(50, 900))
    e = rng.integers(0, n, (int(rng.integers(n, 8 * n)), 2))
    feats = rng.uniform(-1, 2, (n, int(rng.integers(1, 140))))
    nparts = int(rng.integers(1, 9))
    part_of = rng.integers(0, nparts, n)
    part_of[:nparts] = np.arange(nparts)               # every part non-empty
    pick = list(rng.permutation(nparts)[: int(rng.integers(1, nparts + 1))])
    bits = int(rng.integers(1, 9))
    loops = bool(seed % 2)
    g_ours = bg.Graph(n, e, feats)
    g_ref = R.Graph(n, e, feats)
    ours = bg.build_batch(g_ours, bg.PartitionAssignment(nparts, part_of), pick, bg.QuantParams(-1.0, 2.0, bits),
                          add_self_loops=loops)
    ref = R.build_batch(g_ref, R.PartitionAssignment(nparts, part_of), pick, R.QuantParams(-1.0, 2.0, bits),
                        add_self_loops=loops)
    assert np.array_equal(np.asarray(ours.adjacency.words), ref.adjacency.words)
    assert np.array_equal(ours.degrees(), ref.degrees())
    assert bg.pack_batch(ours).data == R.pack_batch(ref).data
