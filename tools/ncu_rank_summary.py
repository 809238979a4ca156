"""Summarise tools/ncu_rank_sweep.sh: per R and kernel family, launches, total time,
time-weighted FP64 tensor-pipe utilisation, DMMA instructions, DRAM bytes."""
import collections
import csv
import re
import sys

for path in sorted(sys.argv[1:], key=lambda p: int(re.search(r"R(\d+)", p).group(1))):
    R = int(re.search(r"R(\d+)", path).group(1))
    rows = [l for l in open(path) if l.startswith('"')]
    L = collections.OrderedDict()
    for r in csv.DictReader(rows):
        try:
            v = float(r["Metric Value"].replace(",", "") or 0)
        except ValueError:
            continue
        L.setdefault((int(r["ID"]), r["Kernel Name"]), {})[r["Metric Name"]] = v
    fam = collections.OrderedDict()
    for (i, k), m in L.items():
        k = re.sub(r"\(.*", "", k).replace("void ", "")
        k = re.sub(r"<.*", "", k).split("::")[-1]
        f = fam.setdefault(k, collections.Counter())
        t = m.get("gpu__time_duration.sum", 0.0) / 1e3
        f["n"] += 1
        f["us"] += t
        f["tensor_us"] += t * m.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0.0)) / 100
        f["dmma"] += m.get("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", 0.0)
        f["dram"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        f["regs"] = max(f["regs"], m.get("launch__registers_per_thread", 0.0))
    for k, f in fam.items():
        tf = f["dmma"] * 512 / (f["us"] * 1e-6) / 1e12 if f["us"] else 0.0
        print(f"R={R:3d} {k:16s} launches {int(f['n']):3d}  {f['us']:9.1f} us  tensor pipe {100 * f['tensor_us'] / max(f['us'], 1e-9):5.1f}%  "
              f"DMMA {f['dmma']:.3g} ({tf:5.1f} TF/s of 37.0 measured)  DRAM {f['dram'] / 1e9:6.3f} GB  regs {int(f['regs'])}")
