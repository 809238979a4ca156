"""One warm config-3 sample call (N = 4, 1.5e7 x 32 fp32-stored, J = 2^20) for ncu."""
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
for i in range(2):
    s.sample_device(None, J, 7 + i, idx, prob, rows)
s.sync()
torch.cuda.profiler.start()
s.sample_device(None, J, 100, idx, prob, rows)
s.sync()
torch.cuda.profiler.stop()
