"""Max CTAs co-resident on one SM during a bmm_reduced launch (C5 shape), from the
per-CTA %globaltimer entry/exit stamps and %smid.   python tools/occupancy_check.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
from c5_sweep import make_operands  # noqa: E402

from paper_2111_09547_b200 import bitgemm, tiled  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
dense, codes, a, x = make_operands(n, 0.1, 4)
tiled.bmm_reduced(a, x)
torch.cuda.synchronize()
rec = []
bitgemm.PHASE_HOOK = rec
tiled.bmm_reduced(a, x)
torch.cuda.synchronize()
bitgemm.PHASE_HOOK = None
st = rec[0][0].cpu().numpy()
st = st[st[:, 0] > 0]
events = []
for row in st:
    events.append((row[0], 1, int(row[6])))
    events.append((row[5], -1, int(row[6])))
events.sort()
cur, best = {}, {}
for t, d, sm in events:
    cur[sm] = cur.get(sm, 0) + d
    best[sm] = max(best.get(sm, 0), cur[sm])
vals = np.array(list(best.values()))
print(f"n={n} pair={tiled.PAIR} ctas={len(st)} SMs used={len(vals)} max co-resident per SM: "
      f"max={vals.max()} mean={vals.mean():.2f}  span={(st[:, 5].max() - st[:, 0].min()) / 1e3:.1f}us")
