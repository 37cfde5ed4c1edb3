"""Timeline of the tiled GEMM launches inside the captured epoch graph (%globaltimer
stamps, L2 flushed before the replay), chained vs two-launch stage pairs.
    python tools/graph_timeline.py [C2] [bits]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_09547_b200 import engine, synth  # noqa: E402
from paper_2111_09547_b200.runtime import EpochRunner  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = synth.with_bits(synth.CONFIGS[name], bits)
batches, feats, _ = synth.planted_batches(cfg, seed=0)
model = synth.calibrated_model(cfg, batches[0], feats[0])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for chain in (True, False):
    engine.CHAIN = chain
    r = EpochRunner(model, batches, rescan=False).capture(stamps=True)
    acc = None
    reps = 20
    for i in range(reps + 3):
        flush.zero_()
        r.run()
        torch.cuda.synchronize()
        if i < 3:
            continue
        rows = []
        for st, _ in r.stamps:
            s = st.cpu().numpy().astype(np.float64)
            s = s[s[:, 0] > 0]
            d = np.diff(s[:, :6], axis=1)
            rows.append([s[:, 0].min(), s[:, 0].max(), s[:, 5].max(), len(s), d[:, 0].mean(), d[:, 1].mean(),
                         d[:, 2].mean(), d[:, 3].mean()])
        rows = np.array(rows)
        rows[:, :3] -= rows[0, 0]
        acc = rows if acc is None else acc + rows
    acc /= reps
    print(f"chain={int(chain)}  (us; mean of {reps} replays)")
    for i, (a, b, c, n, su, ft, ml, ep) in enumerate(acc):
        print(f"  launch {i}: ctas={int(n)} first-start {a / 1e3:6.2f} last-start {b / 1e3:6.2f} end {c / 1e3:6.2f}"
              f" | per-CTA setup {su / 1e3:.2f} first-tile {ft / 1e3:.2f} mainloop {ml / 1e3:.2f} epilogue {ep / 1e3:.2f}")
