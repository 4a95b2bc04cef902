"""Summarise an `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
--csv` log into per-kernel averages and merge them into profiles/ncu_traffic.json under a
config key (bench.py reads roofline.traffic from it).

    python tools/ncu_traffic.py <ncu.csv> <key, e.g. n262144_nb512_t8> [profiles/ncu_traffic.json]
"""
import collections
import csv
import json
import os
import re
import sys

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6,
         "ms": 1e-3, "s": 1.0}


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr, recs = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            recs.append(dict(zip(hdr, r)))
    per = collections.defaultdict(dict)  # launch id -> metrics
    names = {}
    for d in recs:
        lid = d["ID"]
        m = re.search(r"(\w+_kernel)", d["Kernel Name"])
        names[lid] = m.group(1) if m else d["Kernel Name"][:40]
        per[lid][d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
    # split a kernel's launches by grid size when recorded (bulk vs panel-column updates)
    for lid, ms in per.items():
        # tc2_update_kernel serves both the bulk and the panel-column update: split by
        # grid; the co-scheduled tc2w bulk kernel has a per-step grid, keep it whole
        if "launch__grid_size" in ms and names[lid].startswith("tc2_update_kernel"):
            names[lid] += f"[grid={int(ms['launch__grid_size'])}]"
        # tcf_update_kernel: panel-column updates run on 64 CTAs (option 4), the
        # co-scheduled bulk updates on a per-step grid > 64
        elif "launch__grid_size" in ms and names[lid].startswith("tcf_update_kernel"):
            names[lid] += "[pcol]" if int(ms["launch__grid_size"]) <= 64 else "[bulk]"
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for lid, ms in per.items():
        a = agg[names[lid]]
        a[0] += 1
        a[1] += ms.get("dram__bytes_read.sum", 0.0) + ms.get("dram__bytes_write.sum", 0.0)
        a[2] += ms.get("gpu__time_duration.sum", 0.0)
    return {k: {"launches": v[0], "dram_bytes_per_launch": v[1] / v[0],
                "avg_duration_ms": v[2] / v[0] * 1e3,
                "dram_gbs": v[1] / v[2] / 1e9 if v[2] else None} for k, v in agg.items()}


if __name__ == "__main__":
    out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
    cur = json.load(open(out)) if os.path.exists(out) else {}
    cur[sys.argv[2]] = summarise(sys.argv[1])
    json.dump(cur, open(out, "w"), indent=1, sort_keys=True)
    print(json.dumps(cur[sys.argv[2]], indent=1))
