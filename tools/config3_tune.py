"""Config-3 sample call (N = 4, 1.5e7 x 32 fp32-stored, J = 2^20) under tuning options: device ms per call."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2301_12584_b200 import KrpSampler  # noqa: E402

N, I, R, J = 4, 15_000_000, 32, 1 << 20
g = torch.Generator(device="cuda").manual_seed(3)
fs = [torch.rand(I, R, dtype=torch.float32, device="cuda", generator=g) * 2 - 1 for _ in range(N)]
s = KrpSampler.from_device(fs, storage="f32")
del fs
idx = torch.empty(J, N, dtype=torch.int32, device="cuda")
prob = torch.empty(J, dtype=torch.float64, device="cuda")
rows = torch.empty(J, R, dtype=torch.float64, device="cuda")
stream = torch.cuda.ExternalStream(s.stream(), device="cuda")
base = None
for opts in ({}, {"deep_chunk": 0},
             {"deep_threshold": 16}, {"deep_threshold": 32}):
    s.set_tuning(**opts)
    ts = []
    for i in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        s.sample_device(None, J, 100, idx, prob, rows)
        e1.record(stream)
        s.sync()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    same = None
    if base is None:
        base = idx.clone()
    else:
        same = bool(torch.equal(base, idx))
    print(json.dumps({"tuning": opts, "ms": round(min(ts[1:]), 3), "same_indices": same}), flush=True)
