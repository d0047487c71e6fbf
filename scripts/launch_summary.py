"""Summarise an ncu CSV launch list (gpu__time_duration.sum [+ dram__bytes_read/write.sum]):
per-kernel launches, time, share and DRAM bytes; skip the first N launches (warm-up rep).
usage: launch_summary.py launches.csv [skip_first]"""
import csv
import sys

path = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = list(csv.reader(open(path)))
hdr = None
per = {}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = (d["ID"], d["Kernel Name"])
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    m = per.setdefault(key, {})
    if d["Metric Name"] == "gpu__time_duration.sum":
        m["ms"] = v / 1e6 if u in ("nsecond", "ns") else v / 1e3 if u in ("usecond", "us") else v
    elif d["Metric Name"].startswith("dram__bytes"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
        m["dram"] = m.get("dram", 0.0) + v * scale
launches = sorted(per.items(), key=lambda kv: int(kv[0][0]))[skip:]
agg = {}
for (i, k), m in launches:
    k = k.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("nrt::", "")[:50]
    a = agg.setdefault(k, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += m.get("ms", 0.0)
    a[2] += m.get("dram", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"# {len(launches)} launches, {tot:.1f} ms total (cold-cache serialised: compare SHARES)")
print(f"{'kernel':50s} {'launches':>8s} {'ms':>9s} {'share':>6s} {'DRAM GB':>9s} {'TB/s':>6s}")
for k, (n, ms, dr) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:50s} {n:8d} {ms:9.2f} {100 * ms / tot:5.1f}% {dr / 1e9:9.2f} {dr / 1e9 / max(ms, 1e-9):6.2f}")
