"""Where the time of the host API sample() goes (config 2): output allocation, the C call
(setup + kernels + D2H), the Python wrapping."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import make_factors  # noqa: E402
from paper_2301_12584_b200 import KrpSampler  # noqa: E402
from paper_2301_12584_b200 import sampler as smod  # noqa: E402


class A:
    N, I, R, seed = 3, 1 << 22, 64, 2301


def main():
    fs = make_factors(A(), "cuda")
    s = KrpSampler.from_device(fs)
    J = 65536
    for i in range(3):
        s.sample(None, J, i)
    ts = {"alloc": [], "call": [], "total": []}
    for i in range(8):
        t0 = time.perf_counter()
        idx = smod._host_array((J, 3), np.uint32)
        prob = smod._host_array((J,), np.float64)
        rows = smod._host_array((J, 64), np.float64)
        t1 = time.perf_counter()
        import ctypes as C
        smod.check(smod._lib.lib().krpg_sample(s._h, -1, J, 100 + i, 0, 0, idx.ctypes.data_as(C.POINTER(C.c_uint32)),
                                               smod._ptr(prob), smod._ptr(rows), None))
        t2 = time.perf_counter()
        b = s.sample(None, J, 200 + i)
        t3 = time.perf_counter()
        ts["alloc"].append(t1 - t0)
        ts["call"].append(t2 - t1)
        ts["total"].append(t3 - t2)
        del b
    idxd = torch.empty(J, 3, dtype=torch.int32, device="cuda")
    probd = torch.empty(J, dtype=torch.float64, device="cuda")
    rowsd = torch.empty(J, 64, dtype=torch.float64, device="cuda")
    dev = []
    for i in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.sample_device(None, J, 300 + i, idxd, probd, rowsd)
        torch.cuda.synchronize()
        dev.append(time.perf_counter() - t0)
    hb = torch.empty(J, 64, dtype=torch.float64, pin_memory=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hb.copy_(rowsd)
    torch.cuda.synchronize()
    d2h = time.perf_counter() - t0
    print({k: f"{np.median(v) * 1e3:.2f} ms" for k, v in ts.items()},
          f"sync sample_device {np.median(dev) * 1e3:.2f} ms, D2H rows {d2h * 1e3:.2f} ms "
          f"({J * 64 * 8 / d2h / 1e9:.1f} GB/s)")


if __name__ == "__main__":
    main()
