"""Build a config's batches, calibrate, capture one epoch graph and time it; optional
oracle parity on sampled parts.  python tools/run_config.py C4 [bits] [max_batches]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_09547_b200 import synth  # noqa: E402
from paper_2111_09547_b200.runtime import EpochRunner  # noqa: E402

name = sys.argv[1]
cfg = synth.CONFIGS[name]
if len(sys.argv) > 2:
    cfg = synth.with_bits(cfg, int(sys.argv[2]))
nb = -(-cfg.num_parts // cfg.parts_per_batch)
limit = int(sys.argv[3]) if len(sys.argv) > 3 else nb
t0 = time.perf_counter()
batches, feats, xp = synth.planted_batches(cfg, seed=0, batch_ids=range(min(nb, limit)))
torch.cuda.synchronize()
t1 = time.perf_counter()
model = synth.calibrated_model(cfg, batches[0], feats[0])
t2 = time.perf_counter()
runner = EpochRunner(model, batches, rescan=False).capture()
torch.cuda.synchronize()
t3 = time.perf_counter()
st = runner.stream
for _ in range(3):
    with torch.cuda.stream(st):
        runner.run()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
reps = 10
with torch.cuda.stream(st):
    ev[0].record(st)
    for _ in range(reps):
        runner.run()
    ev[1].record(st)
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / reps
nodes = sum(b.total_nodes for b in batches)
print(f"{cfg.name}: batches={len(batches)} nodes={nodes} build={t1 - t0:.1f}s calib={t2 - t1:.1f}s "
      f"capture={t3 - t2:.1f}s  epoch={ms:.3f} ms  ({ms * nb / len(batches):.3f} ms full-epoch est)  "
      f"mem={torch.cuda.max_memory_allocated() / 2**30:.1f} GiB")

# per-launch timing of the grouped GEMM stages (events around back-to-back launches)
from paper_2111_09547_b200 import bitgemm, engine  # noqa: E402
rec = []
bitgemm.PROFILE_HOOK = rec
with torch.cuda.stream(st):
    engine.model_forward_group(batches, model)
    torch.cuda.synchronize()
    rec.clear()
    torch.cuda._sleep(int(2e8))
    engine.model_forward_group(batches, model)
    torch.cuda.synchronize()
bitgemm.PROFILE_HOOK = None
peak = 4155.8
for i, (s, e, w) in enumerate(rec):
    t = s.elapsed_time(e)
    print(f"  stage {i}: {t:.3f} ms  work {w / 1e12:.3f} T-int8-ops  -> {w / (t * 1e-3) / 1e12:.1f} TOPS "
          f"({w / (t * 1e-3) / 1e12 / peak:.1%} of int8 peak)")
