"""Run a config's epoch eagerly (individual launches) for ncu launch lists / captures.

    python tools/profile_epoch.py --config C2 --bits 4 --epochs 2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2111_09547_b200 import engine, synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C2")
p.add_argument("--bits", type=int, default=4)
p.add_argument("--epochs", type=int, default=2)
p.add_argument("--batches", type=int, default=0, help="limit the number of batches (0 = all)")
a = p.parse_args()
cfg = synth.with_bits(synth.CONFIGS[a.config], a.bits)
ids = range(a.batches) if a.batches else None
batches, feats, _ = synth.planted_batches(cfg, seed=0, batch_ids=ids)
model = synth.calibrated_model(cfg, batches[0], feats[0])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(a.epochs):
    for b in batches:
        b.adjacency._schedule = None
        engine.model_forward_device(b, model)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done", cfg.name, len(batches))
