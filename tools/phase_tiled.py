"""Per-CTA phase timeline of the tiled GEMM launches of one epoch (%globaltimer stamps):
0 entry, 1 setup done, 2 first K tile landed (MMA thread), 3 accumulator ready,
4 epilogue done, 5 exit, 7 (chained launches) stage-2 accumulator ready.      python tools/phase_tiled.py [C2] [bits]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_09547_b200 import bitgemm, engine, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = synth.with_bits(synth.CONFIGS[name], int(sys.argv[2]) if len(sys.argv) > 2 else 4)
nb = int(sys.argv[3]) if len(sys.argv) > 3 else None
batches, feats, _ = synth.planted_batches(cfg, seed=0, **({"batch_ids": range(nb)} if nb else {}))
model = synth.calibrated_model(cfg, batches[0], feats[0])
for _ in range(3):
    engine.model_forward_group(batches, model)
torch.cuda.synchronize()
rec = []
bitgemm.PHASE_HOOK = rec
engine.model_forward_group(batches, model)
torch.cuda.synchronize()
bitgemm.PHASE_HOOK = None
prev_end = None
for i, (st, _) in enumerate(rec):
    s = st.cpu().numpy().astype(np.float64)
    s = s[s[:, 0] > 0]
    t0 = s[:, 0].min()
    d = np.diff(s[:, :6], axis=1) / 1e3
    print(f"launch {i}: ctas={len(s)} span={(s[:, 5].max() - t0) / 1e3:.2f}us  last-start={(s[:, 0].max() - t0) / 1e3:.2f}us"
          f"  per-CTA mean(max) us: setup {d[:, 0].mean():.2f}({d[:, 0].max():.2f})"
          f"  first-tile {d[:, 1].mean():.2f}({d[:, 1].max():.2f})  mainloop {d[:, 2].mean():.2f}({d[:, 2].max():.2f})"
          f"  epilogue {d[:, 3].mean():.2f}({d[:, 3].max():.2f})  teardown {d[:, 4].mean():.2f}({d[:, 4].max():.2f})"
          + (f"  gap-from-prev {(t0 - prev_end) / 1e3:.2f}us" if prev_end is not None else ""))
    if (s[:, 7] > 0).all():
        # chained launch: stamp 7 = stage-2 accumulator ready (after epilogue 1 + stage-2 MMAs)
        e1 = (s[:, 7] - s[:, 3]) / 1e3
        e2 = (s[:, 4] - s[:, 7]) / 1e3
        print(f"          chained: epilogue-1 + stage-2 MMA {e1.mean():.2f}({e1.max():.2f})"
              f"  epilogue-2 {e2.mean():.2f}({e2.max():.2f})")
    prev_end = s[:, 5].max()
