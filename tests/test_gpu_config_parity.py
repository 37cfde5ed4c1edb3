"""Config-scale parity: the production (grouped, tiled) engine vs the REAL reference.

For every BASELINE config the logits of our GPU forward over real-size batches
are compared bit for bit (fp64 ``array_equal``) with ``bitgnn.model_forward`` of
the reference staged unmodified in ``oracle/_ref`` (oracle/make_ref.py),
evaluated on the reference's own ``build_batch`` of the same planted parts and
with the model calibrated by the reference's own ``calibrate_model``.  Batches
are block-diagonal and every term of the layer forward is row-local, so each
part is run through the reference as a one-part batch and compared with its rows
of our batch (oracle/ref_inputs.py).  Without a staged reference the check falls
back to the numpy oracle port (oracle/qgtc_oracle.py) on the same part.

Cases (SURVEY.md section 8 shorthand): C1 full at 2 bits; C2 full at 1, 4 and 8
bits; C3 (4-bit GCN) the first and the last batch in full; C4 (8-bit GIN
hidden 256) three parts of batch 0 and the last part of the last batch.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

CASES = {
    "C1-2bit": ("C1", 2, None),
    "C2-1bit": ("C2", 1, None),
    "C2-4bit": ("C2", 4, None),
    "C2-8bit": ("C2", 8, None),
    "C3-4bit": ("C3", 4, "first_last_batches"),
    "C4-8bit": ("C4", 8, [(0, 0), (0, 3), (0, 7), ("last", "last")]),
}

_MODELS = {}


def _worker_logits(job):
    """Reference (or oracle-port) logits of one part; runs in a spawned CPU worker."""
    name, bits, b, p = job
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    from threadpoolctl import threadpool_limits

    import ref_inputs
    from paper_2111_09547_b200 import synth_host as H
    cfg = H.with_bits(H.CONFIGS[name], bits)
    R = ref_inputs.ref_module()
    with threadpool_limits(1):
        if R is not None:
            key = (name, bits)
            if key not in _MODELS:
                _MODELS[key] = ref_inputs.ref_model(R, cfg, 0)
            out, lo, hi = ref_inputs.ref_part_logits(R, _MODELS[key], cfg, 0, b, p)
            return b, p, lo, hi, out, "reference"
    return b, p, None, None, None, "unavailable"


def _oracle_part(model, cfg, b, p):
    """Fallback checker: the numpy oracle port on the same part (our calibrated model)."""
    import qgtc_oracle as O

    from paper_2111_09547_b200 import synth_host as H
    edges, bnd, x = H.host_batch(cfg, 0, b)
    lo, hi = int(bnd[p]), int(bnd[p + 1])
    n = hi - lo
    el = H.batch_edge_list([edges[p]], np.array([0, n]))
    dense = np.zeros((n, n), dtype=np.uint8)
    dense[el[:, 0], el[:, 1]] = 1
    aw, pr, pc = O.pack_words(dense, O.COL, 8)
    codes = O.quantize_codes(np.asarray(x[lo:hi], dtype=np.float64), 0.0, 1.0, cfg.bits)
    from paper_2111_09547_b200.quantize import QuantParams
    return O.model_forward(aw, (n, n, pr, pc), codes, QuantParams(0.0, 1.0, cfg.bits), model.layers), lo, hi


@pytest.mark.gpu
@pytest.mark.parametrize("case", list(CASES))
def test_config_scale_logits_match_reference(case):
    import torch

    from paper_2111_09547_b200 import synth_host as H
    from paper_2111_09547_b200.engine import model_forward_group
    from paper_2111_09547_b200.synth import calibrated_model, planted_batches
    name, bits, sel = CASES[case]
    cfg = H.with_bits(H.CONFIGS[name], bits)
    nb = H.num_batches(cfg)
    sizes = H.batch_part_sizes(cfg)
    if sel is None:
        parts = [(b, p) for b in range(nb) for p in range(len(sizes[b]))]
    elif sel == "first_last_batches":
        parts = [(b, p) for b in (0, nb - 1) for p in range(len(sizes[b]))]
    else:
        parts = [(nb - 1 if b == "last" else b, len(sizes[nb - 1]) - 1 if p == "last" else p) for b, p in sel]
    bids = sorted({b for b, _ in parts})

    # the production path: calibrate on global batch 0, grouped tiled epoch over the batches
    b0, f0, _ = planted_batches(cfg, seed=0, batch_ids=[0])
    model = calibrated_model(cfg, b0[0], f0[0], seed=0)
    batches, _, _ = planted_batches(cfg, seed=0, batch_ids=bids)
    outs = model_forward_group(batches, model)
    torch.cuda.synchronize()
    ours = {b: o.cpu().numpy() for b, o in zip(bids, outs)}

    jobs = [(name, bits, b, p) for b, p in parts]
    with mp.get_context("spawn").Pool(min(len(jobs), os.cpu_count() or 1)) as pool:
        results = pool.map(_worker_logits, jobs, chunksize=max(1, len(jobs) // (os.cpu_count() or 1)))
    kinds = set()
    checked = 0
    for b, p, lo, hi, want, kind in results:
        if kind == "unavailable":
            want, lo, hi = _oracle_part(model, cfg, b, p)
            kind = "oracle-port"
        kinds.add(kind)
        got = ours[b][lo:hi]
        assert got.shape == want.shape
        assert np.array_equal(got, want), f"{case}: batch {b} part {p} rows [{lo},{hi}) differ ({kind})"
        checked += hi - lo
    print(f"{case}: {len(parts)} parts, {checked} nodes bit-exact vs {sorted(kinds)}")
