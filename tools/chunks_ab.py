"""e2e runner time vs the number of pipelined batch chunks.
    python tools/chunks_ab.py [C3] [bits] [chunks,...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_09547_b200 import synth  # noqa: E402
from paper_2111_09547_b200.runtime import HostEpochRunner  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ks = [int(k) for k in (sys.argv[3] if len(sys.argv) > 3 else "8,12,16,24").split(",")]
cfg = synth.with_bits(synth.CONFIGS[name], bits)
batches, feats, _ = synth.planted_batches(cfg, seed=0)
model = synth.calibrated_model(cfg, batches[0], feats[0])
ref = None
for k in ks:
    h = HostEpochRunner(model, batches, chunks=k)
    st = h.stream
    for _ in range(3):
        out = h.run_host()
        st.synchronize()
    if ref is None:
        ref = out.clone()
    same = torch.equal(out, ref)
    n = 20
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = 0.0
    for _ in range(n):
        s.record(st)
        h.run_host()
        e.record(st)
        st.synchronize()
        tot += s.elapsed_time(e)
    print(f"{name} chunks={h.chunks}: e2e {tot / n:.3f} ms  equal={same}", flush=True)
    del h
    torch.cuda.empty_cache()
