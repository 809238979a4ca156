"""CP-ARLS-LEV product sampler (sketch.cpp:86-149) at the headline
shape: N=3 factors 2^22 x 64 (config-2 inputs: N(0,1), 1% of rows Pareto(1.5)-scaled),
J = 65536 draws per call. One call = the reference's whole function: per included factor
G = gram(U), pinv, all I leverage scores, the cumulative table, then the J draws,
probabilities and rows (host outputs).

Device: krpg_product_lev_sample over resident factors (cached Grams) and the free
function krpg_product_lev_sample_factors (host factors: H2D + gram on device).
Reference: its own product_lev_sample (oracle/_ref, all host cores) on a bounded sample
(--ref-rows rows per factor; the per-call cost is dominated by O(I R^2) work, linear in I).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2301_12584_b200 import KrpSampler, product_lev_sample  # noqa: E402


def factors(N, I, R, seed, dev):
    fs = []
    for k in range(N):
        g = torch.Generator(device=dev).manual_seed(seed * 1000 + k)
        U = torch.randn(I, R, dtype=torch.float64, device=dev, generator=g)
        u = torch.rand(I, dtype=torch.float64, device=dev, generator=g)
        w = torch.pow(1.0 - torch.rand(I, dtype=torch.float64, device=dev, generator=g), -1.0 / 1.5)
        U *= torch.where(u < 0.01, w, torch.ones_like(w))[:, None]
        fs.append(U)
    return fs


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--N", type=int, default=3)
    p.add_argument("--I", type=int, default=1 << 22)
    p.add_argument("--R", type=int, default=64)
    p.add_argument("--J", type=int, default=65536)
    p.add_argument("--reps", type=int, default=10)
    p.add_argument("--ref-rows", type=int, default=1 << 19)
    p.add_argument("--no-ref", action="store_true")
    a = p.parse_args()
    dev = torch.device("cuda:0")
    fs = factors(a.N, a.I, a.R, 2301, dev)
    s = KrpSampler.from_device(fs, device=0)
    for _ in range(2):
        s.product_lev_sample(None, a.J, 1)
    ts = []
    for i in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.product_lev_sample(None, a.J, 100 + i)
        ts.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.median(ts))
    # leverage kernel alone (one factor, device events on the sampler's stream)
    stream = torch.cuda.ExternalStream(s.stream(), device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.leverage_scores(0)
    torch.cuda.synchronize()
    e0.record(stream)
    s.leverage_scores(0)
    e1.record(stream)
    torch.cuda.synchronize()
    lev_call_ms = e0.elapsed_time(e1)
    out = {"what": "cp_arls_lev_product_sample", "N": a.N, "I": a.I, "R": a.R, "J": a.J,
           "handle_ms_per_call": ms, "handle_samples_per_s": a.J / (ms / 1e3),
           "leverage_scores_call_ms_incl_d2h": lev_call_ms,
           "u_bytes_per_factor": a.I * a.R * 8}
    host = [f.cpu().numpy() for f in fs]
    del fs
    torch.cuda.empty_cache()
    tf = []
    for i in range(3):
        t0 = time.perf_counter()
        product_lev_sample(host, None, a.J, 200 + i)
        tf.append(time.perf_counter() - t0)
    out["free_function_ms_per_call"] = 1e3 * float(np.median(tf))
    if not a.no_ref:
        import oracle
        if oracle.ref_available():
            sub = [h[: a.ref_rows] for h in host]
            t0 = time.perf_counter()
            oracle.backend("ref").product_lev_sample(sub, None, a.J, 7)
            dt = time.perf_counter() - t0
            out["reference"] = {"rows_per_factor": a.ref_rows, "s_per_call": dt, "cores": os.cpu_count(),
                                "s_per_call_scaled_to_I": dt * a.I / a.ref_rows,
                                "note": "reference product_lev_sample (oracle/_ref) on the first ref_rows rows; "
                                        "cost is O(I R^2) in the table build, scaled linearly to I"}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
