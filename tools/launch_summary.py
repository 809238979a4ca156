"""Summarise an ncu --csv launch list: per-kernel count, time, DRAM bytes.
usage: python tools/launch_summary.py launches.csv [--last-call]"""
import collections
import csv
import re
import sys


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    L = collections.OrderedDict()
    for r in rows:
        k = (int(r["ID"]), r["Kernel Name"])
        L.setdefault(k, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", "") or 0)
    return L


def short(n):
    n = re.sub(r"\(.*", "", n)
    n = re.sub(r"^void ", "", n)
    n = re.sub(r"krpg::(v2::)?(\(anonymous namespace\)::)?", "", n)
    return n[:60]


def main():
    L = load(sys.argv[1])
    items = list(L.items())
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
    for (i, n), m in items:
        a = agg[short(n)]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0)
        a[2] += m.get("dram__bytes_read.sum", 0)
        a[3] += m.get("dram__bytes_write.sum", 0)
        a[4] += m.get("smsp__inst_executed.sum", 0)
    tot = sum(v[1] for v in agg.values())
    print(f"{len(items)} launches, {tot/1e6:.3f} ms total")
    for k, (c, t, r, w, ins) in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
        print(f"{c:6d} {t/1e6:9.3f} ms {100*t/tot:5.1f}%  rd {r/1e9:7.3f} GB  wr {w/1e9:7.3f} GB  inst {ins/1e6:9.1f}M  {k}")


if __name__ == "__main__":
    main()
