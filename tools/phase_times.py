"""Per-phase CTA timing of the bit-GEMM launches of one epoch (globaltimer stamps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_09547_b200 import bitgemm, engine, synth  # noqa: E402

cfg = synth.with_bits(synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"], 4)
batches, feats, _ = synth.planted_batches(cfg, seed=0, batch_ids=[0])
model = synth.calibrated_model(cfg, batches[0], feats[0])
for _ in range(3):
    engine.model_forward_device(batches[0], model)
torch.cuda.synchronize()
rec = []
bitgemm.PHASE_HOOK = rec
engine.model_forward_device(batches[0], model)
torch.cuda.synchronize()
bitgemm.PHASE_HOOK = None
names = ["setup", "mainloop", "epi-compute", "store", "teardown"]
for i, st in enumerate(rec):
    full = st.cpu().numpy()
    full = full[full[:, 0] > 0]
    s = full[:, :6]
    t0 = s[:, 0].min()
    span = (s[:, 5].max() - t0) / 1e3
    start = (s[:, 0] - t0) / 1e3
    cyc = np.diff(s[:, 1:5], axis=1)          # clock64 cycles between stamps 1..4
    names = ["mainloop", "epi-compute", "store"]
    print(f"launch {i}: ctas={len(s)} span={span:.1f}us start(max)={start.max():.1f}us  total(ns)="
          f"{np.mean(s[:, 5] - s[:, 0]):.0f}  "
          + "  ".join(f"{n}={cyc[:, k].mean():.0f}/{cyc[:, k].max():.0f}cyc" for k, n in enumerate(names)))
    # main-loop iteration timeline of the slowest CTA (sync'd, mma-wait done, expanded, issued)
    slow = full[np.argmax(full[:, 5] - full[:, 0])]
    its = slow[6:].reshape(16, 4)
    its = its[its[:, 0] > 0]
    if len(its):
        base = slow[1]
        print("   slowest CTA iterations (cycles from setup: synced,mma-waited,expanded,issued): " + " | ".join(
            f"{r[0]-base},{r[1]-base},{r[2]-base},{r[3]-base}" for r in its[:8]))
    dbg = slow[54:62]
    if dbg.any():
        print("   iteration-1 per-warp cycles (expand, fence):", [(int(x // 100000), int(x % 100000)) for x in dbg])
