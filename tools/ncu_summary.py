"""Summarise an `ncu --set full` capture of one slice per kernel family:
launches, duration, DRAM bytes read/written (the `traffic` the bench reports).

    ncu -i gpurun_out/x.ncu-rep --page raw --csv > x.csv
    python tools/ncu_summary.py x.csv --config c2 --alg-json prof.json [--update profiles/ncu_traffic.json]
"""
import argparse
import collections
import csv
import json
import re


def family(name):
    m = re.search(r"tc::(k_[a-z_]+)", name) or re.search(r"(k_[a-z_]+)", name)
    return m.group(1) if m else name.split("(")[0][:40]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--config", required=True)
    ap.add_argument("--update", default=None)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    hdr = rows[0]
    units = rows[1]
    col = {h: i for i, h in enumerate(hdr)}

    def val(r, key):
        i = col.get(key)
        if i is None or not r[i]:
            return 0.0
        x = float(r[i].replace(",", ""))
        u = units[i]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(u, 1)
        return x * scale

    fam = collections.defaultdict(lambda: dict(launches=0, ns=0.0, rd=0.0, wr=0.0))
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        f = family(r[col["Kernel Name"]])
        e = fam[f]
        e["launches"] += 1
        e["ns"] += val(r, "gpu__time_duration.sum")
        e["rd"] += val(r, "dram__bytes_read.sum")
        e["wr"] += val(r, "dram__bytes_write.sum")
    out = {}
    for f, e in sorted(fam.items(), key=lambda x: -x[1]["ns"]):
        gbs = (e["rd"] + e["wr"]) / e["ns"] if e["ns"] else 0.0
        print(f"{f:22s} launches={e['launches']:5d} time_ms={e['ns'] / 1e6:9.3f} dram_read_GB={e['rd'] / 1e9:8.3f} "
              f"dram_write_GB={e['wr'] / 1e9:8.3f} dram_GB/s={gbs:8.1f}")
        out[f] = dict(launches=e["launches"], time_ms_cold=e["ns"] / 1e6, dram_read=int(e["rd"]),
                      dram_write=int(e["wr"]), dram_bytes_per_slice=int(e["rd"] + e["wr"]),
                      scope=f"all {e['launches']} {f} launches of one {a.config} slice, ncu --set full "
                            f"--clock-control none (serialised, cold); {a.note}")
    if a.update:
        try:
            d = json.load(open(a.update))
        except FileNotFoundError:
            d = {}
        d[a.config] = out
        json.dump(d, open(a.update, "w"), indent=1)


if __name__ == "__main__":
    main()
