"""One grouped epoch (all batches per launch, as in the bench's graph) run eagerly after
two warm-up epochs, bracketed by cudaProfilerStart/Stop for ncu --profile-from-start off.

    ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,\
dram__bytes_write.sum --clock-control none --csv --log-file X.csv python tools/ncu_epoch.py C4 8
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_09547_b200 import engine, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = synth.with_bits(synth.CONFIGS[name], int(sys.argv[2]) if len(sys.argv) > 2 else 8)
batches, feats, _ = synth.planted_batches(cfg, seed=0)
model = synth.calibrated_model(cfg, batches[0], feats[0])
for _ in range(2):
    engine.model_forward_group(batches, model)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
engine.model_forward_group(batches, model)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done", cfg.name, len(batches))
