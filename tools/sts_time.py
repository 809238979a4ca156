import sys, os, time, json, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from paper_2301_12584_b200 import KrpSampler, SparseTensor
from parity_util import sparse_tensor
dims, R = (4_800_000, 1_800_000, 1_800_000), 64
coords, values = sparse_tensor(dims, int(os.environ.get("STS_NNZ", "20000000")), seed=5)
T = SparseTensor(dims, coords, values)
g = torch.Generator(device="cuda").manual_seed(1)
fs = [torch.randn(d, R, dtype=torch.float64, device="cuda", generator=g) for d in dims]
s = KrpSampler.from_device(fs)
for j in range(3): s.sts_solve(T, j, 65536, j)
s.profile_enable(True)
for j in range(3):
    s.profile_read(reset=True); torch.cuda.synchronize(); t0=time.perf_counter()
    s.sts_solve(T, j, 65536, 10 + j); torch.cuda.synchronize(); w=time.perf_counter()-t0
    pr = s.profile_read(reset=True)
    print(j, round(w*1e3,2), {k: round(v["ms"],3) for k,v in pr.items() if v["launches"]}, s.sts_last_stats())
