"""A/B of chained vs two-launch stage pairs, device epoch graph and e2e runner, in one
process (alternating rounds).     python tools/chain_ab.py [C3] [bits] [rounds]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_09547_b200 import engine, synth  # noqa: E402
from paper_2111_09547_b200.runtime import EpochRunner, HostEpochRunner  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 4
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = synth.with_bits(synth.CONFIGS[name], bits)
batches, feats, _ = synth.planted_batches(cfg, seed=0)
model = synth.calibrated_model(cfg, batches[0], feats[0])
runners = {}
for chain in (True, False):
    engine.CHAIN = chain
    runners[chain] = (EpochRunner(model, batches, rescan=False).capture(), HostEpochRunner(model, batches))
engine.CHAIN = True
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def t_dev(r, n=50):
    st = torch.cuda.current_stream()
    tot = 0.0
    for i in range(n + 5):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(st)
        r.run()
        e.record(st)
        torch.cuda.synchronize()
        if i >= 5:
            tot += s.elapsed_time(e)
    return tot / n


def t_e2e(h, n=30):
    st = h.stream
    tot = 0.0
    for i in range(n + 3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(st)
        out = h.run_host()
        e.record(st)
        st.synchronize()
        _ = float(out[0, 0])
        if i >= 3:
            tot += s.elapsed_time(e)
    return tot / n


a = runners[True][1].run_host()
runners[True][1].stream.synchronize()
b = runners[False][1].run_host()
runners[False][1].stream.synchronize()
same = torch.equal(a, b)
print(f"{name} bits={bits} chunks={runners[True][1].chunks} e2e outputs equal: {same}")
for rnd in range(rounds):
    for chain in (True, False):
        d, h = runners[chain]
        print(f"round {rnd} chain={int(chain)}: device {t_dev(d):.4f} ms  e2e {t_e2e(h):.4f} ms")
