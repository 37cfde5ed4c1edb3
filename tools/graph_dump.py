"""Dump the node/edge structure of the captured C2 epoch graph (DOT, verbose) and list
its nodes in order with their kinds; shows whether kernel->kernel edges are
programmatic (PDL) edges.     python tools/graph_dump.py [C2] [out.dot]"""
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_09547_b200 import synth  # noqa: E402
from paper_2111_09547_b200.runtime import EpochRunner  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/graph.dot"
cfg = synth.with_bits(synth.CONFIGS[name], 4)
batches, feats, _ = synth.planted_batches(cfg, seed=0)
model = synth.calibrated_model(cfg, batches[0], feats[0])
r = EpochRunner(model, batches, rescan=False)
orig = torch.cuda.CUDAGraph


class DebugGraph(orig):
    def __init__(self, *a, **k):
        k.setdefault("keep_graph", True)
        super().__init__(*a, **k)
        self.enable_debug_mode()


torch.cuda.CUDAGraph = DebugGraph
try:
    r.capture()
finally:
    torch.cuda.CUDAGraph = orig
r.graph.debug_dump(out)
txt = open(out).read()
for line in txt.splitlines():
    if "->" in line or "KERNEL" in line or "MEMSET" in line or "MEMCPY" in line or "label" in line[:200]:
        pass
kinds = re.findall(r'(KERNEL|MEMSET|MEMCPY|EVENT_RECORD|WAIT_EVENT|EMPTY|HOST)', txt)
print("node kinds:", {k: kinds.count(k) for k in set(kinds)})
edges = [l.strip() for l in txt.splitlines() if "->" in l]
print(len(edges), "edges")
for e in edges[:40]:
    print(" ", e[:200])
names = re.findall(r'\\n(_Z[^\\]*|[a-z_]+kernel[^\\]*)\\n', txt)
print("kernels:", [n[:60] for n in names][:40])
