"""One config-4 point for ncu: N = 3 factors 2^20 x R (N(0,1)), one tree rebuild of
factor 0 and one sample(nullopt, J = 65536). Usage: python tools/rank_point.py R"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2301_12584_b200 import KrpSampler  # noqa: E402

R = int(sys.argv[1])
g = torch.Generator(device="cuda").manual_seed(R)
fs = [torch.randn(1 << 20, R, dtype=torch.float64, device="cuda", generator=g) for _ in range(3)]
s = KrpSampler.from_device(fs)
s.sample(None, 65536, 1)  # warm (setup cache, buffers)
s.rebuild(0)
s.sample(None, 65536, 2)
s.sync()
