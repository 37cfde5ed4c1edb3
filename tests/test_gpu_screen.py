"""The tiled epilogue's fp32 requant screen (csrc/qgtc_tiled.cu, ScreenRow) against
the oracle on adversarial grids.

With weight and feature grids starting at 0 and no bias, the dequantized value is
k_acc * acc exactly and a power-of-two output scale puts the requant quotient
acc * 2^-j EXACTLY on code boundaries for many elements: every such element must
leave the screen and take the exact fp64 path.  Logits must equal the oracle's bit
for bit (fp64).  The config-scale tests (test_gpu_config_parity.py) cover random
grids.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2111_09547_b200 as bg
from oracle import qgtc_oracle as O
from paper_2111_09547_b200 import engine, synth

pytestmark = pytest.mark.gpu


def _boundary_model(kind: str, in_dim: int, classes: int, hidden: int, bits: int, e: int):
    build = engine.gcn_model if kind == "gcn" else engine.gin_model
    model = build(in_dim, classes, hidden_dim=hidden, num_layers=3, feature_bits=bits, weight_bits=bits, seed=3,
                  weight_range=(0.0, 1.0), with_bias=False)
    for layer in model.layers:
        # scale = 2^(e - bits): quotients are dyadic multiples of the accumulator
        layer.mid_params = bg.QuantParams(0.0, 2.0 ** e, bits)
        if layer.output_mode == "bitplanes":
            layer.out_params = bg.QuantParams(0.0, 2.0 ** (e + 2), bits)
    model._prepared = None
    return model


@pytest.mark.parametrize("kind", ["gcn", "gin"])
@pytest.mark.parametrize("bits,e", [(8, -4), (8, 0), (8, 4), (4, 0), (4, 3), (2, 1)])
def test_screen_on_exact_code_boundaries(kind, bits, e):
    cfg = synth.GraphConfig("screen", kind, 700, 9000, 4, 4, 40, 32, 10, 3, bits, bits)
    batches, feats, xp = synth.planted_batches(cfg, seed=5)
    b = batches[0]
    model = _boundary_model(kind, cfg.in_dim, cfg.classes, cfg.hidden, bits, e)
    got = bg.model_forward(b, model)
    a = b.adjacency
    codes = O.quantize_codes(feats[0], xp.alpha_min, xp.alpha_max, xp.bits)
    want = O.model_forward(a.words, a.dims(), codes, xp, model.layers)
    assert got.shape == want.shape
    assert np.array_equal(got, want)


def test_screen_matches_random_grids_wide():
    # hidden 256 (bn = 256 tiles, chained GIN stages) with calibrated (random) grids
    cfg = synth.GraphConfig("screen-wide", "gin", 900, 12000, 3, 3, 100, 256, 47, 3, 8, 8)
    batches, feats, xp = synth.planted_batches(cfg, seed=9)
    b = batches[0]
    model = synth.calibrated_model(cfg, b, feats[0], seed=9)
    got = bg.model_forward(b, model)
    a = b.adjacency
    codes = O.quantize_codes(feats[0], xp.alpha_min, xp.alpha_max, xp.bits)
    want = O.model_forward(a.words, a.dims(), codes, xp, model.layers)
    assert np.array_equal(got, want)
