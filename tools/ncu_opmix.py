"""Instruction mix + top stall lines of kernel block k of an ncu report's SASS source page.
    python tools/ncu_opmix.py report.ncu-rep [k] [ntop]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for ln in out.split("\n"):
    if ln.startswith('"Kernel Name"'):
        cur = []
        blocks.append((ln, cur))
    elif cur is not None and ln.strip():
        cur.append(ln)
name, body = blocks[k]
rows = list(csv.reader(body))
hdr, data = rows[0], [r for r in rows[1:] if len(r) == len(rows[0])]
idx = {h: i for i, h in enumerate(hdr)}
ie, st = "Instructions Executed", "Warp Stall Sampling (All Samples)"
tot = sum(float(r[idx[ie]] or 0) for r in data)
tots = sum(float(r[idx[st]] or 0) for r in data)
ops = collections.Counter()
for r in data:
    t = r[idx["Source"]].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    ops[op.split(".")[0]] += float(r[idx[ie]] or 0)
print(name[:90], f"| {len(blocks)} blocks | warp-instr {int(tot)} | samples {int(tots)}")
print("op mix: " + ", ".join(f"{o}={v / tot:.1%}" for o, v in ops.most_common(18)))
top = sorted(range(len(data)), key=lambda j: -float(data[j][idx[st]] or 0))[:ntop]
for j in sorted(top):
    r = data[j]
    print(f"{j:5d} {float(r[idx[st]]) / tots:5.1%} x{r[idx[ie]]:>8s}  {r[idx['Source']].strip()[:80]}")
