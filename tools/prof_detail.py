"""Per-kernel-type device time of one sample() on config 2 (warm, events on the stream)."""
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
    if len(sys.argv) > 1:
        a.I = int(sys.argv[1])
    if len(sys.argv) > 2:
        a.R = int(sys.argv[2])
    fs = make_factors(a, "cuda")
    s = KrpSampler.from_device(fs)
    J = 65536
    idx = torch.empty(J, 3, dtype=torch.int32, device="cuda")
    prob = torch.empty(J, dtype=torch.float64, device="cuda")
    rows = torch.empty(J, a.R, dtype=torch.float64, device="cuda")
    for i in range(3):
        s.sample_device(None, J, i, idx, prob, rows)
    s.profile_enable(True, detail=True)
    s.profile_read(reset=True)
    K = 5
    for i in range(K):
        s.sample_device(None, J, 100 + i, idx, prob, rows)
    p = s.profile_read(reset=True)
    tot = 0
    for k, v in p.items():
        if v["ms"] > 0 or v["launches"]:
            print(f"  {k:14s} {v['ms'] / K:8.3f} ms/step  launches/step {v['launches'] / K:6.1f}")


if __name__ == "__main__":
    main()
