"""Top stall lines of an ncu report's SASS source page (needs -lineinfo + --import-source)."""
import csv
import subprocess
import sys

rep, k = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for ln in out.split("\n"):
    if ln.startswith('"Kernel Name"'):
        cur = []
        blocks.append((ln, cur))
        continue
    if cur is not None and ln.strip():
        cur.append(ln)
name, body = blocks[k]
rows = list(csv.reader(body))
hdr = rows[0]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[1:]
ie, st = "Instructions Executed", "Warp Stall Sampling (All Samples)"
tot_i = sum(float(r[idx[ie]] or 0) for r in data)
tot_s = sum(float(r[idx[st]] or 0) for r in data)
print(name[:100], "| warp-instr", int(tot_i), "| samples", int(tot_s), "| sass lines", len(data))
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {h: sum(float(r[idx[h]] or 0) for r in data) for h in reasons}
print("stall mix:", ", ".join(f"{k[6:]}={v / tot_s:.0%}" for v, k in sorted(((v, k) for k, v in agg.items()),
                                                                        reverse=True)[:7]))
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
top = sorted(range(len(data)), key=lambda j: -float(data[j][idx[st]] or 0))[:n]
for j in sorted(top):
    r = data[j]
    rs = sorted(((float(r[idx[h]] or 0), h[6:]) for h in reasons), reverse=True)[:2]
    print(f"{j:5d} {float(r[idx[st]]) / tot_s:5.1%} x{r[idx[ie]]:>7s}  {r[idx['Source']][:72]:72s} {rs}")
