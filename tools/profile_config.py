"""One eager grouped forward of a config (for ncu): python tools/profile_config.py C4 8 [batches]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_09547_b200 import engine, synth  # noqa: E402
from paper_2111_09547_b200.tiled import blocked, weight_tiles  # noqa: E402

cfg = synth.with_bits(synth.CONFIGS[sys.argv[1]], int(sys.argv[2]))
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 16
batches, feats, _ = synth.planted_batches(cfg, seed=0, batch_ids=range(nb))
model = synth.calibrated_model(cfg, batches[0], feats[0])
for b in batches:
    blocked(b.adjacency)
for ly, prep in zip(model.layers, engine._prepared(model)):
    weight_tiles(ly, prep)
engine.model_forward_group(batches, model)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
engine.model_forward_group(batches, model)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
