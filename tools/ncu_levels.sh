#!/bin/bash
# warm per-launch device times of one sample() (ncu, --cache-control none: no flush between kernels)
# usage: tools/ncu_levels.sh out.csv [env assignments...]
out=$1; shift
env "$@" ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum --cache-control none --clock-control none -k regex:"k_eval|k_deep2|k_make_z|k_stage|k_apply|k_etree" -s 140 -c 66 --csv --log-file $out python tools/prof_detail.py > /dev/null 2>&1
python - $out <<'PY'
import csv, re, sys, collections
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
L = collections.OrderedDict()
for r in csv.DictReader(lines):
    L.setdefault((int(r["ID"]), r["Kernel Name"]), {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", "") or 0)
tot = collections.Counter(); n = collections.Counter()
for (i, k), m in L.items():
    k = re.sub(r"\(.*", "", k).replace("void ", "")
    tot[k] += m["gpu__time_duration.sum"] / 1e3; n[k] += 1
    print("%3d %-28s %8.1f us  tensor %5.1f%%  dram %6.1f MB" % (i, k[:28], m["gpu__time_duration.sum"] / 1e3, m["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"], m["dram__bytes_read.sum"] / 1e6))
print("totals (ms):", {k: (round(v / 1e3, 3), n[k]) for k, v in tot.items()})
PY
