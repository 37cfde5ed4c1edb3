"""Host-side inputs for the REAL reference -- TEST / BASELINE INFRASTRUCTURE ONLY.

Builds the reference's own objects for the synthetic configs without touching
this package's kernels: the planted graph comes from the numpy-only generator
``paper_2111_09547_b200.synth_host`` (the same stream the GPU path consumes),
batches from the reference's ``build_batch`` (graph.py:308-357), models from
the reference presets (engine.py:408-453, same seed => same weights) calibrated
by the reference's ``calibrate_model`` on global batch 0 (engine.py:372-405,
cli.py:209).  Users: ``tests/`` (config-scale parity) and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (HERE, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)


def ref_module():
    """The staged real reference (oracle/_ref/bitgnn), or None when not staged."""
    import make_ref
    if not make_ref.available():
        return None
    return make_ref.import_reference()


def ref_build(R, cfg, edges, boundaries, x):
    """Reference build_batch over the parts in ``edges`` (their own graph: cross-part
    edges are dropped by build_batch anyway, graph.py:337)."""
    from paper_2111_09547_b200 import synth_host as H
    total = int(boundaries[-1])
    el = H.batch_edge_list(edges, boundaries, self_loops=False)
    g = R.Graph(total, el, features=np.asarray(x, dtype=np.float64))
    part_of = np.repeat(np.arange(len(boundaries) - 1), np.diff(boundaries))
    assign = R.PartitionAssignment(len(boundaries) - 1, part_of)
    return R.build_batch(g, assign, list(range(len(boundaries) - 1)), R.QuantParams(0.0, 1.0, cfg.bits))


def ref_model(R, cfg, seed):
    """Reference preset calibrated on the reference-built global batch 0."""
    from paper_2111_09547_b200 import synth_host as H
    builder = R.gcn_model if cfg.model == "gcn" else R.gin_model
    model = builder(cfg.in_dim, cfg.classes, hidden_dim=cfg.hidden, num_layers=cfg.layers,
                    feature_bits=cfg.bits, weight_bits=cfg.wbits, seed=seed)
    edges, bnd, x = H.host_batch(cfg, seed, 0)
    b0 = ref_build(R, cfg, edges, bnd, x)
    R.calibrate_model(model, b0, np.asarray(x, dtype=np.float64))
    return model


def ref_part_batch(R, cfg, seed, b, p):
    """Part p of batch b as a one-part reference SubgraphBatch, plus its batch-local
    row range [lo, hi).  Batches are block-diagonal and every term of the layer
    forward is row-local, so the part's logits equal those rows of the batch's."""
    from paper_2111_09547_b200 import synth_host as H
    edges, bnd, x = H.host_batch(cfg, seed, b)
    lo, hi = int(bnd[p]), int(bnd[p + 1])
    return ref_build(R, cfg, [edges[p]], np.array([0, hi - lo]), x[lo:hi]), lo, hi


def ref_part_logits(R, model, cfg, seed, b, p):
    rb, lo, hi = ref_part_batch(R, cfg, seed, b, p)
    return R.model_forward(rb, model), lo, hi
