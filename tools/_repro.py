import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2111_09547_b200 as bg
from paper_2111_09547_b200 import synth, engine
from oracle import qgtc_oracle as O
mode = sys.argv[1]
bits = 4
cfg = synth.GraphConfig("boundary", "gin", 700, 6000, 4, 4, 40, 24, 7, 3, bits, bits)
batches, feats, xp = synth.planted_batches(cfg, seed=3)
model = synth.calibrated_model(cfg, batches[0], feats[0], seed=3)
if mode.startswith("int"):
    rng = np.random.default_rng(bits)
    for ly in model.layers:
        ly.weight = rng.integers(0, 1 << bits, ly.weight.shape).astype(np.float64)
        ly.weight_params = bg.QuantParams(0.0, float(1 << bits), bits)
        if ly.bias is not None:
            ly.bias = rng.integers(-3, 4, ly.bias.shape).astype(np.float64)
        for name in ("mid_params", "out_params"):
            if getattr(ly, name) is not None:
                setattr(ly, name, bg.QuantParams(0.0, float(1 << bits), bits))
    model._prepared = None
engine.SCREEN = mode.endswith("screen")
out = engine.model_forward_group(batches, model)[0].cpu().numpy()
a = batches[0].adjacency
codes = O.quantize_codes(feats[0], xp.alpha_min, xp.alpha_max, xp.bits)
want = O.model_forward(a.words, a.dims(), codes, xp, model.layers)
print(mode, "fused" if engine.FUSED_EPOCH else "staged", "OK" if np.array_equal(out, want) else "MISMATCH")
