"""Host-side cost of one asynchronous sample_device call (R x R setup + enqueue) vs its
device time, per rank R (config 4 shapes)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2301_12584_b200 import KrpSampler  # noqa: E402


def main():
    for R in (64, 128, 256):
        g = torch.Generator(device="cuda").manual_seed(R)
        fs = [torch.randn(1 << 20, R, dtype=torch.float64, device="cuda", generator=g) for _ in range(3)]
        s = KrpSampler.from_device(fs)
        del fs
        J = 65536
        idx = torch.empty(J, 3, dtype=torch.int32, device="cuda")
        prob = torch.empty(J, dtype=torch.float64, device="cuda")
        rows = torch.empty(J, R, dtype=torch.float64, device="cuda")
        for i in range(2):
            s.sample_device(None, J, i, idx, prob, rows)
        torch.cuda.synchronize()
        # host time of a synchronous call's setup ~ async call return time when the GPU is idle
        s.set_async(True)
        t0 = time.perf_counter()
        s.sample_device(None, J, 50, idx, prob, rows)
        t_enq = time.perf_counter() - t0
        s.sync()
        t_all = time.perf_counter() - t0
        K = 6
        t0 = time.perf_counter()
        for i in range(K):
            s.sample_device(None, J, 60 + i, idx, prob, rows)
        s.sync()
        t_k = (time.perf_counter() - t0) / K
        s.set_async(False)
        print(f"R={R}: enqueue (host setup) {t_enq * 1e3:.1f} ms, single call {t_all * 1e3:.1f} ms, "
              f"pipelined {t_k * 1e3:.1f} ms/call", flush=True)
        s.close()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
