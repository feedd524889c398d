"""Sum ncu dram__bytes_read.sum + dram__bytes_write.sum over all kernels of a CSV
(ncu --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum), and per kernel name."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot = collections.defaultdict(float)
per = collections.defaultdict(lambda: collections.defaultdict(float))
ids = set()
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    m = d.get("Metric Name")
    if m not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        continue
    unit = d.get("Metric Unit", "byte")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
    v = float(d["Metric Value"].replace(",", "")) * scale
    tot[m] += v
    ids.add(d.get("ID"))
    per[re.sub(r"\(.*", "", d["Kernel Name"])][m] += v
print(f"launches {len(ids)} read {tot['dram__bytes_read.sum'] / 1e9:.3f} GB write {tot['dram__bytes_write.sum'] / 1e9:.3f} GB "
      f"total {(tot['dram__bytes_read.sum'] + tot['dram__bytes_write.sum']) / 1e9:.3f} GB")
for k, d in sorted(per.items(), key=lambda x: -sum(x[1].values()))[:15]:
    print(f"  {sum(d.values()) / 1e9:8.3f} GB  {k[:100]}")
