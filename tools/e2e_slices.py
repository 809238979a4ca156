"""e2e (host outputs through KrpSampler.sample) vs the number of output slices of the
last position (KRPG_OPT_OUT_SLICES), config 2. One JSON line per setting."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from bench import make_factors  # noqa: E402
from paper_2301_12584_b200 import KrpSampler  # noqa: E402


class A:
    N, I, R, seed = 3, 1 << 22, 64, 2301


s = KrpSampler.from_device(make_factors(A(), "cuda"))
J = 65536
for so in (1, 2, 3, 4):
    s.set_tuning(out_slices=so)
    for i in range(3):
        s.sample(None, J, 7 + i)
    ts = []
    for i in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.sample(None, J, 100 + i)
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(json.dumps({"out_slices": so, "median_ms": 1e3 * ts[len(ts) // 2], "min_ms": 1e3 * ts[0],
                      "samples_per_s_median": J / ts[len(ts) // 2]}), flush=True)
