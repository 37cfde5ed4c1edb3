"""Dump the node list of the captured C2 epoch graph (kernel names / memsets / memcpys)."""
import os
import re
import sys
from collections import Counter

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_09547_b200 import synth  # noqa: E402
from paper_2111_09547_b200.runtime import EpochRunner  # noqa: E402

cfg = synth.with_bits(synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"], 4)
batches, feats, _ = synth.planted_batches(cfg, seed=0)
model = synth.calibrated_model(cfg, batches[0], feats[0])
orig = torch.cuda.CUDAGraph.__init__


def init(self, *a, **k):
    orig(self, *a, **k)
    self.enable_debug_mode()


torch.cuda.CUDAGraph.__init__ = init
r = EpochRunner(model, batches, rescan=False).capture()
path = "gpurun_out/epoch_graph.dot"
r.graph.debug_dump(path)
text = open(path).read()
kinds = Counter()
for m in re.finditer(r'label="\{([A-Z_]+)[^|]*\|([^}]*)', text):
    kind, rest = m.group(1), m.group(2)
    name = re.search(r"(qg::\w+|at::\w+|\w+_kernel\w*|cudaMemset|memset|memcpy)", rest)
    kinds[(kind, name.group(1) if name else rest[:40])] += 1
for (k, n), c in sorted(kinds.items()):
    print(f"{c:3d}  {k:12s} {n}")
