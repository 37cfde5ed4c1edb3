"""Why is a cold (L2-flushed) C2 epoch slower than a warm one?  Times the epoch graph
warm, after a 256 MB flush (bench style), and the per-launch GEMM durations after a flush.

    python tools/cold_step.py [C2] [bits]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_09547_b200 import bitgemm, engine, synth  # noqa: E402
from paper_2111_09547_b200.runtime import EpochRunner  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = synth.with_bits(synth.CONFIGS[name], bits)
batches, feats, _ = synth.planted_batches(cfg, seed=0)
model = synth.calibrated_model(cfg, batches[0], feats[0])
r = EpochRunner(model, batches, rescan=False).capture()
st = r.stream
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
small = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def steps(n, pre=None, sync=False):
    ev = []
    with torch.cuda.stream(st):
        for _ in range(n):
            if pre is not None:
                pre()
            if sync:
                torch.cuda.synchronize()
            s, e = E(), E()
            s.record(st)
            r.run()
            e.record(st)
            ev.append((s, e))
    torch.cuda.synchronize()
    return sum(s.elapsed_time(e) for s, e in ev) / n * 1e3


steps(10)
print(f"{cfg.name} {bits}-bit epoch graph (us):")
print(f"  warm back-to-back          {steps(50):8.1f}")
print(f"  after 256MB write flush    {steps(50, lambda: flush.zero_()):8.1f}")
print(f"  flush + host sync          {steps(50, lambda: flush.zero_(), True):8.1f}")
print(f"  after 256MB read (sum)     {steps(50, lambda: small.sum()):8.1f}")
print(f"  after 16MB write           {steps(50, lambda: flush[:16 << 20].zero_()):8.1f}")
print(f"  after 64MB write           {steps(50, lambda: flush[:64 << 20].zero_()):8.1f}")

rec = []
bitgemm.PROFILE_HOOK = rec
with torch.cuda.stream(st):
    for cold in (False, True):
        engine.model_forward_group(batches, model)
        torch.cuda.synchronize()
        rec.clear()
        if cold:
            flush.zero_()
        torch.cuda._sleep(int(2e8))
        engine.model_forward_group(batches, model)
        torch.cuda.synchronize()
        print(("cold" if cold else "warm") + " per-launch GEMM us: " +
              " ".join(f"{s.elapsed_time(e) * 1e3:.1f}" for s, e, _ in rec))
bitgemm.PROFILE_HOOK = None
