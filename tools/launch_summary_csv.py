"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) by kernel."""
import collections
import csv
import re
import sys

rows = [l for l in open(sys.argv[1]) if l.startswith('"')]
L = collections.OrderedDict()
for r in csv.DictReader(rows):
    try:
        v = float(r["Metric Value"].replace(",", "") or 0)
    except ValueError:
        continue
    L.setdefault((int(r["ID"]), r["Kernel Name"]), {})[r["Metric Name"]] = v
tot = collections.Counter()
n = collections.Counter()
dr = collections.Counter()
for (i, k), m in L.items():
    k = re.sub(r"\(.*", "", k).replace("void ", "")
    tot[k] += m.get("gpu__time_duration.sum", 0) / 1e3
    dr[k] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    n[k] += 1
T = sum(tot.values())
print(f"{len(L)} launches, {T / 1e3:.3f} ms serialised")
for k, v in tot.most_common():
    print(f"  {k[:60]:60s} {n[k]:4d} x  {v / 1e3:8.3f} ms  ({100 * v / T:5.1f} %)  DRAM {dr[k] / 1e9:7.3f} GB")
