"""Break the e2e epoch (bench.py `e2e`) into H2D / graph / D2H with CUDA events.

    python tools/e2e_breakdown.py [C2] [bits]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_09547_b200 import synth  # noqa: E402
from paper_2111_09547_b200.runtime import EpochRunner, HostEpochRunner  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = synth.with_bits(synth.CONFIGS[name], bits)
batches, feats, _ = synth.planted_batches(cfg, seed=0)
model = synth.calibrated_model(cfg, batches[0], feats[0])
host = HostEpochRunner(model, batches)
dev = EpochRunner(model, batches, rescan=False).capture()
st = host.stream
reps = 50


def timed(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        s.record(st)
        for _ in range(reps):
            fn()
        e.record(st)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def h2d():
    with torch.cuda.stream(st):
        host.device.copy_(host.host, non_blocking=True)


def graph_rescan():
    with torch.cuda.stream(st):
        host.inner.run()


def graph_static():
    with torch.cuda.stream(dev.stream):
        dev.run()


outs = host.inner.logits


def d2h():
    with torch.cuda.stream(st):
        r = 0
        for o in outs:
            host.out_host[r:r + o.shape[0]].copy_(o, non_blocking=True)
            r += o.shape[0]


def full():
    host.run_host()


print(f"{cfg.name} {bits}-bit: H2D {host.h2d_bytes / 1e6:.2f} MB, D2H {host.d2h_bytes / 1e6:.2f} MB")
for nm, fn in (("h2d", h2d), ("graph (rescan)", graph_rescan), ("graph (static)", graph_static), ("d2h", d2h),
               ("e2e run_host", full)):
    print(f"  {nm:16s} {timed(fn) * 1e3:9.1f} us")
