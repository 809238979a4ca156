"""Where does the host-API (e2e) time go? sample() with different output buffers."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from bench import make_factors  # noqa: E402
from paper_2301_12584_b200 import KrpSampler, _lib  # noqa: E402


class A:
    N, I, R, seed = 3, 1 << 22, 64, 2301


def main():
    a = A()
    fs = make_factors(a, "cuda")
    s = KrpSampler.from_device(fs)
    J, N, R = 65536, 3, 64
    L = _lib.lib()
    dp = C.POINTER(C.c_double)

    def raw(idx, prob, rows, tag):
        ts = []
        for i in range(6):
            t0 = time.perf_counter()
            _lib.check(L.krpg_sample(s.handle, -1, J, 100 + i, 0, 0, idx.ctypes.data_as(C.POINTER(C.c_uint32)),
                                     prob.ctypes.data_as(dp), rows.ctypes.data_as(dp), None))
            ts.append(time.perf_counter() - t0)
        print(f"{tag:28s} median {1e3*np.median(ts[1:]):7.2f} ms  ({J/np.median(ts[1:]):.3e}/s)")

    raw(np.empty((J, N), np.uint32), np.empty(J), np.empty((J, R)), "pageable reused")
    ts = []
    for i in range(6):
        t0 = time.perf_counter()
        s.sample(None, J, 200 + i)
        ts.append(time.perf_counter() - t0)
    print(f"{'sample() fresh arrays':28s} median {1e3*np.median(ts[1:]):7.2f} ms")
    pi = torch.empty((J, N), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    pp = torch.empty(J, dtype=torch.float64, pin_memory=True).numpy()
    pr = torch.empty((J, R), dtype=torch.float64, pin_memory=True).numpy()
    raw(pi, pp, pr, "pinned reused")
    idx = torch.empty(J, N, dtype=torch.int32, device="cuda")
    prob = torch.empty(J, dtype=torch.float64, device="cuda")
    rows = torch.empty(J, R, dtype=torch.float64, device="cuda")
    ts = []
    for i in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.sample_device(None, J, 300 + i, idx, prob, rows)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{'device outputs (wall)':28s} median {1e3*np.median(ts[1:]):7.2f} ms")


if __name__ == "__main__":
    main()
