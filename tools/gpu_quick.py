"""Quick GPU correctness/timing probe used during development (not a test)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))

import oracle  # noqa: E402
from parity_util import compare_draws, pareto_factors, rel_err_matrix, rel_err_vec, rows_rel_err  # noqa: E402
from paper_2301_12584_b200 import KrpSampler  # noqa: E402


def check_trees(shapes, seed):
    fs = pareto_factors(shapes, seed)
    s = KrpSampler(fs)
    o = oracle.OracleKrp(fs, "port")
    worst = 0.0
    for j, f in enumerate(fs):
        L, n = s.tree_shape(j)
        for v in [0] + list(range(1, n, 2)):
            worst = max(worst, rel_err_matrix(s.node_gram(j, v), o.node_gram(j, v)))
    print(f"trees {shapes}: worst node rel err {worst:.2e}")
    return s, o, fs


def check_sample(s, o, J, seed, mode="two_stage"):
    for e in [None] + list(range(s.factor_count())):
        t0 = time.time()
        b = s.sample(e, J, seed, mode=mode, margin=True)
        t1 = time.time()
        ri, rp, rr, rm = o.sample(e, J, seed, one_stage=(mode == "one_stage"), want_margin=True)
        n, nb, nu = compare_draws(b.indices, b.margin, ri, rm)
        ok = nu == 0
        same = ~np.any(b.indices != ri, axis=1)
        pe = rel_err_vec(b.probabilities[same], rp[same])
        re = rows_rel_err(b.rows[same], rr[same])
        print(f"  {mode} excl={e}: mismatches {n} (boundary {nb}, unexplained {nu}) prob rel {pe:.1e} rows rel {re:.1e} gpu {t1-t0:.3f}s {'OK' if ok else 'FAIL'}")


def main():
    for shapes in [[(8, 3), (7, 3), (6, 3)], [(64, 4), (40, 4), (33, 4)], [(4096, 16)] * 3,
                   [(1000, 8), (777, 8), (513, 8)], [(5000, 64), (3000, 64), (4097, 64)],
                   [(300, 5), (200, 5)], [(2000, 32), (1500, 32), (999, 32), (1234, 32)]]:
        s, o, fs = check_trees(shapes, 1)
        check_sample(s, o, 4096, 7)
        check_sample(s, o, 4096, 7, mode="one_stage")
    # timing at a larger size
    import torch
    for I, R in [(1 << 20, 64), (1 << 22, 64)]:
        g = torch.Generator(device="cuda").manual_seed(0)
        fs = [torch.randn(I, R, dtype=torch.float64, device="cuda", generator=g) for _ in range(3)]
        torch.cuda.synchronize()
        t0 = time.time()
        s = KrpSampler.from_device(fs)
        torch.cuda.synchronize()
        t1 = time.time()
        print(f"I={I} R={R}: build (3 factors) {t1-t0:.3f}s wall, last tree {s.last_build_ms():.3f} ms")
        J = 65536
        idx = torch.empty(J, 3, dtype=torch.int32, device="cuda")
        prob = torch.empty(J, dtype=torch.float64, device="cuda")
        rows = torch.empty(J, R, dtype=torch.float64, device="cuda")
        for it in range(3):
            torch.cuda.synchronize()
            t0 = time.time()
            s.sample_device(None, J, 11 + it, idx, prob, rows)
            torch.cuda.synchronize()
            t1 = time.time()
            print(f"   sample J={J}: {1e3*(t1-t0):.2f} ms -> {J/(t1-t0):.3e} samples/s")
        del s


if __name__ == "__main__":
    main()
