"""From an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,...
--csv), print the 0-based launch index (for ncu --launch-skip, no kernel filter) of the
launch of a kernel family with the most DRAM bytes among launches [first, ...).

    python tools/ncu_pick.py list.csv k_stream_pair [--first 200]
"""
import argparse
import csv

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("kernel")
ap.add_argument("--first", type=int, default=0)
a = ap.parse_args()
rows = [r for r in csv.reader(open(a.csv)) if len(r) > 10]
hdr = rows[0]
by = {}
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if not d["ID"].isdigit():
        continue
    k = int(d["ID"])
    e = by.setdefault(k, {"name": d["Kernel Name"], "bytes": 0.0})
    if d["Metric Name"].startswith("dram__bytes"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(d["Metric Unit"], 1)
        e["bytes"] += float(d["Metric Value"].replace(",", "")) * scale
best = max((k for k, e in by.items() if k >= a.first and a.kernel in e["name"]), key=lambda k: by[k]["bytes"])
print(best)
