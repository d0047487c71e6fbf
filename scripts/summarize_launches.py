"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per-kernel totals."""
import csv
import sys

path = sys.argv[1]
skip_first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = list(csv.reader(open(path)))
hdr = None
launches = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            v = float(d["Metric Value"].replace(",", ""))
            u = d["Metric Unit"]
            v = v / 1e6 if u in ("nsecond", "ns") else v / 1e3 if u in ("usecond", "us") else v
            launches.append((d["ID"], d["Kernel Name"], v))
launches = launches[skip_first:]
agg = {}
for _, k, v in launches:
    k = k.split("(")[0][:70]
    a = agg.setdefault(k, [0.0, 0])
    a[0] += v
    a[1] += 1
tot = sum(a[0] for a in agg.values())
print(f"{len(launches)} launches, {tot:.3f} ms total")
for k, (v, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{v:9.3f} ms {n:5d}x {100 * v / tot:5.1f}%  {k}")
