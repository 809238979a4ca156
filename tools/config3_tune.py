"""A sample call under tuning options: device ms per call (default shape: config 3, N = 4,
1.5e7 x 32 fp32-stored, J = 2^20).  usage: config3_tune.py [N I R J f32|f64]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2301_12584_b200 import KrpSampler  # noqa: E402

N, I, R, J = 4, 15_000_000, 32, 1 << 20
storage = "f32"
if len(sys.argv) > 5:
    N, I, R, J, storage = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
g = torch.Generator(device="cuda").manual_seed(3)
dt = torch.float32 if storage == "f32" else torch.float64
fs = [torch.rand(I, R, dtype=dt, device="cuda", generator=g) * 2 - 1 for _ in range(N)]
s = KrpSampler.from_device(fs, storage=storage)
del fs
idx = torch.empty(J, N, dtype=torch.int32, device="cuda")
prob = torch.empty(J, dtype=torch.float64, device="cuda")
rows = torch.empty(J, R, dtype=torch.float64, device="cuda")
stream = torch.cuda.ExternalStream(s.stream(), device="cuda")
base = None
for opts in ({}, {"deep_threshold": 8}, {"deep_threshold": 16}, {"deep_threshold": 64}, {"deep_threshold": 128},
             {"deep_threshold": 32, "deep_chunk": 16}, {"deep_chunk": 0}):
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
