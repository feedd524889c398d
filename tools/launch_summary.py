"""Aggregate an ncu --metrics gpu__time_duration.sum CSV by kernel name."""
import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum": continue
    name = d["Kernel Name"]
    name = re.sub(r"\(.*", "", name)
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "ns")
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(unit, 1e-6)
    agg[name][0] += 1; agg[name][1] += v * scale
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.3f} ms over {sum(v[0] for v in agg.values())} launches")
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{ms:9.3f} ms {100*ms/tot:5.1f}%  {n:5d}x  {k[:110]}")
