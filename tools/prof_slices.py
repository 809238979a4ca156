"""Step device time (config 2, async issue like bench.py) for 1..3 descent slices."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from bench import make_factors  # noqa: E402
from paper_2301_12584_b200 import KrpSampler  # noqa: E402


class A:
    N, I, R, seed = 3, 1 << 22, 64, 2301


def main():
    a = A()
    fs = make_factors(a, "cuda")
    s = KrpSampler.from_device(fs)
    J = 65536
    idx = torch.empty(J, 3, dtype=torch.int32, device="cuda")
    prob = torch.empty(J, dtype=torch.float64, device="cuda")
    rows = torch.empty(J, a.R, dtype=torch.float64, device="cuda")
    stream = torch.cuda.ExternalStream(s.stream(), device="cuda")
    s.set_async(True)
    for n in (1, 2, 3, 4):
        s.set_slices(n)
        for i in range(3):
            s.sample_device(None, J, i, idx, prob, rows)
        s.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 10
        e0.record(stream)
        for i in range(K):
            s.sample_device(None, J, 100 + i, idx, prob, rows)
        e1.record(stream)
        s.sync()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        print(f"slices {n}: {ms:.3f} ms/step  {J / ms * 1e3:.4g} samples/s", flush=True)


if __name__ == "__main__":
    main()
