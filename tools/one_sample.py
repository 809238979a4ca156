"""One warm config-2 sample call (for ncu captures of the descent kernels)."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from bench import make_factors  # noqa: E402
from paper_2301_12584_b200 import KrpSampler  # noqa: E402


class A:
    N, I, R, seed = 3, 1 << 22, 64, 2301


s = KrpSampler.from_device(make_factors(A(), "cuda"))
idx = torch.empty(65536, 3, dtype=torch.int32, device="cuda")
prob = torch.empty(65536, dtype=torch.float64, device="cuda")
rows = torch.empty(65536, 64, dtype=torch.float64, device="cuda")
for i in range(3):
    s.sample_device(None, 65536, 7 + i, idx, prob, rows)
s.sync()
