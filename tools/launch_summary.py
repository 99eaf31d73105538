"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total/avg device time and share."""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "")[:60]
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
        v *= scale.get(d["Metric Unit"], 1e-3)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values()) or 1.0
    out = []
    for k, (n, us) in agg.items():
        out.append(f"{k:60s} n={n:4d} total={us:9.2f}us avg={us / n:8.2f}us share={us / tot * 100:5.1f}%")
    out.append(f"{'TOTAL':60s}        total={tot:9.2f}us")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
