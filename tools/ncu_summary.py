"""Summarise an ncu metrics log of ONE slice per kernel family: launches,
duration, DRAM bytes read/written -- the `traffic` the bench reports.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file x.csv python tools/one_slice.py c2
    python tools/ncu_summary.py x.csv --config c2 [--update profiles/ncu_traffic.json]

ncu serialises launches and (by default) flushes caches between them, so times
are cold-cache and per-launch DRAM bytes include re-reads an L2-resident
producer->consumer chain would avoid: compare shares and traffic/alg ratios.
"""
import argparse
import collections
import csv
import json
import re

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
         "second": 1e9}


def family(name):
    m = re.search(r"(k_[a-z_]+)", name)
    return m.group(1) if m else name.split("(")[0][:40]


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    per = collections.OrderedDict()
    for r in csv.DictReader(lines[start:]):
        d = per.setdefault(int(r["ID"]), {"name": r["Kernel Name"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1)
    return per


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--config", required=True)
    ap.add_argument("--update", default=None)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    fam = collections.defaultdict(lambda: dict(launches=0, ns=0.0, rd=0.0, wr=0.0))
    for d in load(a.csv).values():
        e = fam[family(d["name"])]
        e["launches"] += 1
        e["ns"] += d.get("gpu__time_duration.sum", 0.0)
        e["rd"] += d.get("dram__bytes_read.sum", 0.0)
        e["wr"] += d.get("dram__bytes_write.sum", 0.0)
    tot = sum(e["ns"] for e in fam.values())
    out = {}
    for f, e in sorted(fam.items(), key=lambda x: -x[1]["ns"]):
        gbs = (e["rd"] + e["wr"]) / e["ns"] if e["ns"] else 0.0
        print(f"{f:18s} launches={e['launches']:5d} time_ms={e['ns'] / 1e6:9.3f} share={e['ns'] / tot:5.3f} "
              f"dram_read_GB={e['rd'] / 1e9:8.3f} dram_write_GB={e['wr'] / 1e9:8.3f} dram_GB/s={gbs:8.1f}")
        out[f] = dict(launches=e["launches"], time_ms_cold=round(e["ns"] / 1e6, 4), share=round(e["ns"] / tot, 4),
                      dram_read=int(e["rd"]), dram_write=int(e["wr"]), dram_bytes_per_slice=int(e["rd"] + e["wr"]),
                      scope=f"all {e['launches']} {f} launches of one {a.config} slice (tools/one_slice.py), "
                            f"ncu --clock-control none, serialised, caches flushed per launch. {a.note}".strip())
    if a.update:
        try:
            d = json.load(open(a.update))
        except FileNotFoundError:
            d = {}
        d[a.config] = out
        json.dump(d, open(a.update, "w"), indent=1)


if __name__ == "__main__":
    main()
