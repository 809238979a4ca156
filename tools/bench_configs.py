"""Secondary BASELINE.json configurations (the headline config 2 is bench.py):

  --config 3 : N=4 factors 1.5e7 x 32, uniform[-1,1], fp32-stored / fp64-accumulated;
               tree build, 2^20 two-stage draws, 10^5 random single-entry updates; under
               torchrun (WORLD_SIZE > 1) the 2^20 draws are sharded over the ranks (strong
               scaling, NCCL, max over ranks).
  --config 4 : rank sweep, N=3 factors 2^20 x R (R in 16..256), N(0,1); J = 65536.
  --config 5 : STS-CP factor updates (krpg_sts_solve) on a synthetic COO tensor with the
               Amazon-Reviews shape 4.8e6 x 1.8e6 x 1.8e6, Zipf(1.1) coordinates per mode,
               lognormal(0,1) values, duplicates summed; R = 64, J = 65536; the full
               1.7e9 raw nonzeros (--nnz), generated and ingested on the device.

One JSON line per measurement. Device times by CUDA events on the sampler's stream.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from bench import descent_bytes, load_peaks  # noqa: E402
from paper_2301_12584_b200 import KrpSampler  # noqa: E402


def timed(fn, stream, reps):
    evs = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        fn()
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def measure(s, N, I, R, J, storage, label, reps=5, extra=None):
    dev = torch.device("cuda")
    stream = torch.cuda.ExternalStream(s.stream(), device=dev)
    peak, _ = load_peaks()
    # tree build (device time of the leaf + level kernels)
    s.profile_enable(True)
    s.profile_read(reset=True)
    for j in range(N):
        s.rebuild(j)
    pb = s.profile_read(reset=True)
    build_ms = (pb["tree_leaf"]["ms"] + pb["tree_levels"]["ms"]) / N
    P = R * (R + 1) // 2
    L = (I + R - 1) // R
    elt = 4 if storage == "f32" else 8
    build_bytes = I * R * elt + L * P * 8
    idx = torch.empty(J, N, dtype=torch.int32, device=dev)
    prob = torch.empty(J, dtype=torch.float64, device=dev)
    rows = torch.empty(J, R, dtype=torch.float64, device=dev)
    # asynchronous issue as in bench.py: a call's host setup overlaps the previous call's kernels
    s.set_async(True)
    for i in range(2):
        s.sample_device(None, J, 7 + i, idx, prob, rows)
    s.sync()
    s.profile_read(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for i in range(reps):
        s.sample_device(None, J, 100 + i, idx, prob, rows)
    e1.record(stream)
    s.sync()
    torch.cuda.synchronize()
    s.set_async(False)
    prof = s.profile_read(reset=True)
    ms = e0.elapsed_time(e1) / reps
    bytes_step, _ = descent_bytes(idx.cpu().numpy().view(np.uint32), [I] * N, R, elt=elt)
    draws_ms = prof["draws"]["ms"] / reps
    line = {"config": label, "N": N, "I": I, "R": R, "J": J, "storage": storage,
            "samples_per_s": J / (ms / 1e3), "ms_per_sample_call": ms,
            "descent": {"alg_bytes": bytes_step, "kernel_ms": draws_ms,
                        "achieved_gbs": bytes_step / (draws_ms / 1e3) / 1e9,
                        "frac_of_hbm": bytes_step / (draws_ms / 1e3) / 1e9 / peak},
            "tree_build": {"ms_per_factor": build_ms, "alg_bytes": build_bytes,
                           "achieved_gbs": build_bytes / (build_ms / 1e3) / 1e9,
                           "gflops": I * R * (R + 1) / (build_ms / 1e3) / 1e9},
            "descent_path": "grouped-dmma" if (R % 8 == 0 and (R <= 160 or (R <= 256 and R % 32 == 0))) else "per-draw"}
    if extra:
        line.update(extra)
    print(json.dumps(line), flush=True)


def config3_sharded(args):
    """Config 3's draws sharded over the ranks of one node (strong scaling: the 2^20 draws of
    one call split into contiguous ranges, draw_offset = range start, trees replicated --
    bit-identical to one call, sharding.shard_range); launch with torchrun (one process per
    GPU, NCCL). Device time of the call per rank, max over ranks."""
    import torch.distributed as dist

    from paper_2301_12584_b200.sharding import shard_range
    world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    N, I, R, J = 4, 15_000_000, 32, 1 << 20
    g = torch.Generator(device="cuda").manual_seed(3)
    fs = [torch.rand(I, R, dtype=torch.float32, device="cuda", generator=g) * 2 - 1 for _ in range(N)]
    s = KrpSampler.from_device(fs, storage="f32", device=local)
    del fs
    torch.cuda.empty_cache()
    start, count = shard_range(J, rank, world)
    idx = torch.empty(count, N, dtype=torch.int32, device="cuda")
    prob = torch.empty(count, dtype=torch.float64, device="cuda")
    rows = torch.empty(count, R, dtype=torch.float64, device="cuda")
    stream = torch.cuda.ExternalStream(s.stream(), device=torch.device("cuda", local))
    for i in range(2):
        s.sample_device(None, count, 7 + i, idx, prob, rows, draw_offset=start)
    s.sync()
    reps = 3
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(reps):
        s.sample_device(None, count, 100 + i, idx, prob, rows, draw_offset=start)
    e1.record(stream)
    s.sync()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / reps], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        ms = float(t.item())
        print(json.dumps({"config": "config3_sharded", "N": N, "I": I, "R": R, "J": J, "ranks": world,
                          "scaling": "strong (J split over the ranks)", "ms_per_call_max_over_ranks": ms,
                          "samples_per_s": J / (ms / 1e3)}), flush=True)
    dist.destroy_process_group()


def config3(args):
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.sharded:
        return config3_sharded(args)
    N, I, R, J = 4, 15_000_000, 32, 1 << 20
    g = torch.Generator(device="cuda").manual_seed(3)
    fs = [torch.rand(I, R, dtype=torch.float32, device="cuda", generator=g) * 2 - 1 for _ in range(N)]
    s = KrpSampler.from_device(fs, storage="f32")
    del fs
    torch.cuda.empty_cache()
    # 10^5 random single-entry updates on factor 0 (one batched call, wall time incl. transfers)
    rng = np.random.default_rng(5)
    n = 100_000
    r = rng.integers(0, I, n).astype(np.uint64)
    c = rng.integers(0, R, n).astype(np.uint32)
    v = rng.uniform(-1, 1, n)
    s.update_factor_entries(0, r[:10], c[:10], v[:10])  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.update_factor_entries(0, r, c, v)
    torch.cuda.synchronize()
    upd_s = time.perf_counter() - t0
    measure(s, N, I, R, J, "f32", "config3", reps=3,
            extra={"updates": {"count": n, "seconds": upd_s, "updates_per_s": n / upd_s}})


def config4(args):
    for R in args.ranks:
        N, I, J = 3, 1 << 20, 65536
        g = torch.Generator(device="cuda").manual_seed(R)
        fs = [torch.randn(I, R, dtype=torch.float64, device="cuda", generator=g) for _ in range(N)]
        s = KrpSampler.from_device(fs)
        del fs
        measure(s, N, I, R, J, "f64", f"config4_R{R}", reps=3)
        s.close()
        torch.cuda.empty_cache()


def zipf_coords(d, n, s, gen, out, chunk=50_000_000):
    """Bounded continuous power law x^-s on [1, d+1) by inverse CDF, floored to a
    rank, then mapped through a random permutation of the mode (GPU); written into
    the int32 column `out` chunk by chunk so 1.7e9 draws need no large temporaries."""
    perm = torch.randperm(d, device="cuda", generator=gen).to(torch.int32)
    a = 1.0 - s
    top = (d + 1.0) ** a - 1.0
    for c0 in range(0, n, chunk):
        m = min(chunk, n - c0)
        u = torch.rand(m, dtype=torch.float64, device="cuda", generator=gen)
        x = (1.0 + u * top) ** (1.0 / a)
        r = torch.clamp(x.floor().to(torch.int64) - 1, 0, d - 1)
        out[c0:c0 + m] = perm[r]
    del perm


def config5(args):
    dims = (4_800_000, 1_800_000, 1_800_000)
    R, J, nnz = 64, 65536, int(args.nnz)
    gen = torch.Generator(device="cuda").manual_seed(5)
    coords = torch.empty(nnz, 3, dtype=torch.int32, device="cuda")
    col = torch.empty(nnz, dtype=torch.int32, device="cuda")
    for m, d in enumerate(dims):
        zipf_coords(d, nnz, 1.1, gen, col)
        coords[:, m] = col
    del col
    values = torch.empty(nnz, dtype=torch.float64, device="cuda")
    for c0 in range(0, nnz, 50_000_000):
        m = min(50_000_000, nnz - c0)
        values[c0:c0 + m] = torch.randn(m, dtype=torch.float64, device="cuda", generator=gen).exp()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    from paper_2301_12584_b200 import SparseTensor
    t0 = time.perf_counter()
    T = SparseTensor.from_device(dims, coords, values)  # device-side dedup + sort, no host staging
    ingest_s = time.perf_counter() - t0
    del coords, values
    torch.cuda.empty_cache()
    fs = [torch.randn(d, R, dtype=torch.float64, device="cuda", generator=gen) for d in dims]
    s = KrpSampler.from_device(fs)
    del fs
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    for j in range(3):  # warm: fiber indexes + buffers
        s.sts_solve(T, j, J, 100 + j)
    warm_s = time.perf_counter() - t0
    s.profile_enable(True)
    res = []
    for det in (1, 0):  # row-ordered bit-reproducible scatter (default), then fp64 atomics
        s.set_tuning(sts_deterministic=det)
        for rnd in range(args.rounds):
            for j in range(3):
                s.profile_read(reset=True)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                s.sts_solve(T, j, J, 1000 * rnd + j)
                torch.cuda.synchronize()
                wall = time.perf_counter() - t0
                pr = s.profile_read(reset=True)
                res.append({"mode": j, "I_j": dims[j], "wall_ms": wall * 1e3, "stats": s.sts_last_stats(),
                            "deterministic": det,
                            "device_ms": {k: round(v["ms"], 4) for k, v in pr.items() if v["launches"]}})
    s.set_tuning(sts_deterministic=1)
    free, total = torch.cuda.mem_get_info()
    for j in range(3):
        walls = [r["wall_ms"] for r in res if r["mode"] == j and r["deterministic"]]
        walls_at = [r["wall_ms"] for r in res if r["mode"] == j and not r["deterministic"]]
        last = [r for r in res if r["mode"] == j and r["deterministic"]][-1]
        print(json.dumps({"config": "config5", "workload": "STS-CP factor update (krpg_sts_solve)",
                          "dims": dims, "R": R, "J": J, "raw_nnz": nnz, "nnz": T.nnz(),
                          "scaled": ("full raw nonzero count 1.7e9" if nnz >= 1_700_000_000 else
                                     f"raw nonzeros {nnz:.3g} instead of 1.7e9") +
                                    " (synthetic Zipf(1.1) tensor, lognormal values; one GPU)",
                          "mode": j, "ms_per_update_median": float(np.median(walls)),
                          "ms_per_update_median_atomic_scatter": float(np.median(walls_at)),
                          "device_ms_breakdown_last": last["device_ms"], "step_stats_last": last["stats"],
                          "ingest_s": ingest_s, "first_solves_incl_fiber_indexes_s": warm_s,
                          "device_mem_used_gb": (total - free) / 1e9}), flush=True)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, choices=[3, 4, 5], required=True)
    p.add_argument("--nnz", type=float, default=1.7e9)
    p.add_argument("--rounds", type=int, default=3)
    p.add_argument("--ranks", type=int, nargs="+", default=[16, 32, 64, 128, 256])
    p.add_argument("--sharded", action="store_true", help="config 3: the sharded (torchrun) path even at one rank")
    args = p.parse_args()
    torch.cuda.init()
    {3: config3, 4: config4, 5: config5}[args.config](args)


if __name__ == "__main__":
    main()
