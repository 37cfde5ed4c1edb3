import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2111_09547_b200 import _native as N
rng = np.random.default_rng(0)
def run(a, b):
    y = 1.0 / b
    ta, tb, ty = (torch.from_numpy(np.ascontiguousarray(v)).cuda() for v in (a, b, y))
    out, ref = torch.empty_like(ta), torch.empty_like(ta)
    N.call("qg_test_div", N.ptr(ta), N.ptr(tb), N.ptr(ty), ta.numel(), N.ptr(out), N.ptr(ref), N.stream())
    return out.cpu().numpy(), ref.cpu().numpy()
for name, a, b in [("simple", rng.uniform(-5, 5, 10), np.full(10, 0.3)),
                   ("wide", rng.standard_normal(200000) * np.exp2(rng.integers(-1060, 1020, 200000).astype(float)),
                    np.abs(rng.standard_normal(200000)) * np.exp2(rng.integers(-1060, 1020, 200000).astype(float)) + 1e-300)]:
    o, r = run(a, b)
    bad = ~((o.view(np.int64) == r.view(np.int64)) | (np.isnan(o) & np.isnan(r)))
    print(name, "mismatches", bad.sum(), "of", len(a))
    for i in np.nonzero(bad)[0][:8]:
        print("  a=%r b=%r out=%r ref=%r q=%r" % (a[i], b[i], o[i], r[i], a[i] / b[i]))
