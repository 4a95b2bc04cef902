"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections, csv, re, sys

def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
             "s": 1e6, "second": 1e6}
    for d in data:
        if d.get("Metric Name", "gpu__time_duration.sum") != "gpu__time_duration.sum":
            continue
        m = re.search(r"(\w+_kernel(?:<[^>]*>)?|\w*elementwise\w*)", d["Kernel Name"])
        name = m.group(1) if m else d["Kernel Name"][:40]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"].replace(",", "")) * scale[d["Metric Unit"]]
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:40s} n={v[0]:5d} total={v[1] / 1e3:9.2f} ms avg={v[1] / v[0]:9.1f} us "
                   f"share={v[1] / tot:.3f}")
    return "\n".join(out)

if __name__ == "__main__":
    print(summarise(sys.argv[1]))
