"""DRAM traffic of the descent kernels of ONE config-2 sample() step.

Run under ncu with --profile-from-start off (the profiled region is exactly one
sample_device call after warm-up):
  ncu --profile-from-start off --cache-control none --clock-control none \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --csv --log-file out.csv python tools/ncu_step_traffic.py
then `python tools/ncu_step_traffic.py --summarize out.csv` writes profiles/ncu_traffic.json."""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run():
    import torch

    from bench import make_factors
    from paper_2301_12584_b200 import KrpSampler

    class A:
        N, I, R, seed = 3, 1 << 22, 64, 2301

    fs = make_factors(A(), "cuda")
    s = KrpSampler.from_device(fs)
    J = 65536
    idx = torch.empty(J, 3, dtype=torch.int32, device="cuda")
    prob = torch.empty(J, dtype=torch.float64, device="cuda")
    rows = torch.empty(J, 64, dtype=torch.float64, device="cuda")
    for i in range(3):
        s.sample_device(None, J, i, idx, prob, rows)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    s.sample_device(None, J, 100, idx, prob, rows)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


def summarize(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        per.setdefault(r[ii], {"k": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    draws = [v for v in per.values() if any(t in v["k"] for t in ("k_eval", "k_deep", "k_apply_pick", "k_stage_init", "k_pos0",
                                                                  "k_make_z", "k_leaf2", "k_scatter"))]
    rd = sum(v.get("dram__bytes_read.sum", 0) for v in draws)
    wr = sum(v.get("dram__bytes_write.sum", 0) for v in draws)
    ms = sum(v.get("gpu__time_duration.sum", 0) for v in draws) / 1e6
    out = {"draws_bytes_per_step": rd + wr, "read": rd, "write": wr, "kernels": len(draws),
           "serialized_kernel_ms": ms,
           "note": "one config-2 sample() step under ncu --cache-control none (L2 state carried between "
                   "kernels as in a real run), DRAM bytes summed over the descent kernels; "
                   "tools/ncu_step_traffic.py"}
    json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--summarize":
        summarize(sys.argv[2])
    else:
        run()
