"""DRAM traffic per tiled-GEMM launch from an ncu launch list with dram counters
(``ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
-k regex:tc_tiled ... --csv --log-file X.csv python bench.py ...``) into
profiles/ncu_summary.json under "<workload>:bitgemm_dram_bytes_per_launch" (the bench
line's roofline.traffic) plus the per-launch list.

    python tools/ncu_traffic.py gpurun_out/r03a_c4_launches.csv C4-gin-products-2.4M [launches per epoch]
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path, workload = sys.argv[1], sys.argv[2]
per_epoch = int(sys.argv[3]) if len(sys.argv) > 3 else 4
recs, order, hdr = {}, [], None
for r in csv.reader(open(path)):
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    if "tc_tiled" not in d["Kernel Name"] and "tc_pair" not in d["Kernel Name"]:
        continue
    if d["ID"] not in recs:
        order.append(d["ID"])
    recs.setdefault(d["ID"], {"kernel": d["Kernel Name"].split("(")[0]})[d["Metric Name"]] = float(
        d["Metric Value"].replace(",", ""))
launches = [recs[i] for i in order][:per_epoch]
per = [x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in launches]
out_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
summary = json.load(open(out_path)) if os.path.exists(out_path) else {}
summary[f"{workload}:bitgemm_dram_bytes_per_launch"] = sum(per) / len(per)
summary[f"{workload}:per_launch"] = [{"kernel": x["kernel"], "dram_bytes": p,
                                      "ncu_us": x["gpu__time_duration.sum"] / 1e3} for x, p in zip(launches, per)]
summary[f"{workload}:source"] = (f"{os.path.relpath(path, ROOT)} (ncu --metrics dram__bytes_read/write.sum, "
                                 "cold L2 per launch, one epoch)")
json.dump(summary, open(out_path, "w"), indent=1)
print(json.dumps({k: v for k, v in summary.items() if k.startswith(workload)}, indent=1))
