"""Grouped (node-sorted DMMA) vs per-draw descent per rank, config-4 shape
(N = 3 factors 2^20 x R, N(0,1), J = 65536): device time of one sample call each,
and whether both give identical indices (they use different summation orders, so
only boundary draws may differ)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2301_12584_b200 import KrpSampler  # noqa: E402

J = 65536
for R in [int(x) for x in (sys.argv[1:] or ["8", "16", "24", "32", "48", "64"])]:
    g = torch.Generator(device="cuda").manual_seed(R)
    fs = [torch.randn(1 << 20, R, dtype=torch.float64, device="cuda", generator=g) for _ in range(3)]
    s = KrpSampler.from_device(fs)
    del fs
    st = torch.cuda.ExternalStream(s.stream(), device="cuda")
    idx = torch.empty(J, 3, dtype=torch.int32, device="cuda")
    prob = torch.empty(J, dtype=torch.float64, device="cuda")
    rows = torch.empty(J, R, dtype=torch.float64, device="cuda")
    res = {"R": R}
    outs = {}
    for name, grouped in (("grouped", True), ("per_draw", False)):
        s.set_grouped_descent(grouped)
        for i in range(2):
            s.sample_device(None, J, 5 + i, idx, prob, rows)
        s.sync()
        ts = []
        for i in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            s.sample_device(None, J, 100 + i, idx, prob, rows)
            e1.record(st)
            s.sync()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[name + "_ms"] = float(np.median(ts))
        outs[name] = idx.cpu().numpy().copy()
    res["index_mismatches"] = int(np.any(outs["grouped"] != outs["per_draw"], axis=1).sum())
    print(json.dumps(res), flush=True)
    s.close()
    torch.cuda.empty_cache()
