#!/usr/bin/env python
"""bench.py — KRP leverage samples/sec on BASELINE.json config 2.

Workload (config 2): N = 3 dense fp64 factors of shape 2^22 x 64, i.i.d.
N(0,1) entries with 1% of rows scaled by a Pareto(alpha=1.5) weight; one
"step" = KrpSampler::sample(nullopt, J = 65536, seed) — the two-stage draw of
the reference (krp_sampler.cpp:82-151): per-call R x R setup, eigenvector-tree
construction and batched root-to-leaf descent for every factor, probability
epilogue. Factors and trees are resident in HBM before timing starts.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (one process per GPU over NCCL; `--gpus N` without torchrun's
WORLD_SIZE re-executes itself under torch.distributed.run): the tree structure is
replicated and each rank draws its own J with draw ids offset by rank*J (weak
scaling, no collective on the data path); time = max over ranks. At N > 1 the
row-partitioned construction (per-rank subtrees + NCCL all-gather of
level slices and subtree roots) is timed next to "all-gather U + redundant
rebuild" and reported under "construction".

Parity of the benchmarked call itself: rank 0 at N = 1 runs the unmodified
reference (oracle/_ref, the cpu_baseline leg) on the same factors and seeds as
the last timed step and the three exclude-one calls, and reports the comparison
under "parity" (indices bit-exact except counted boundary draws, whose margin
|cutoff - u| <= 1e-10 comes from a deterministic re-run of the same call with
margins; probabilities / rows relative error).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "KRP leverage samples/sec (N=3, I_j=2^22, R=64, fp64)"
WORKLOAD = ("config2: N=3 fp64 factors 2^22x64, N(0,1), 1% rows x Pareto(1.5); "
            "step = sample(nullopt, J=65536) two-stage per rank")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--mode", default="two_stage", choices=["two_stage", "one_stage"])
    p.add_argument("--I", type=int, default=1 << 22)
    p.add_argument("--R", type=int, default=64)
    p.add_argument("--N", type=int, default=3)
    p.add_argument("--J", type=int, default=65536)
    p.add_argument("--seed", type=int, default=2301)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--tune", nargs="*", default=[], metavar="KEY=VALUE",
                   help="kernel-variant / tuning options for A/B runs (KrpSampler.set_tuning keys)")
    return p.parse_args()


REF_FLAGS = ("g++ -std=c++20 -O3 -march=x86-64-v3 -ffp-contract=off -fopenmp (oracle/Makefile; the "
             "reference's own CMake Release build uses -O3 without -march)")


def bench_config(args, world):
    """The workload dict, identical in both arms (the driver compares them)."""
    return {"workload": WORKLOAD, "N": args.N, "I": args.I, "R": args.R, "J": args.J, "mode": args.mode,
            "l2": "flushed (256 MiB write) before every step inside the timed region; resident inputs "
                  "9.7 GB >> L2",
            "parallelism": f"draws sharded across {world} GPU(s) (weak), trees replicated"}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------- inputs
def make_factors(args, device):
    """Seeded synthetic config-2 factors generated on the GPU (Philox)."""
    import torch
    fs = []
    for k in range(args.N):
        g = torch.Generator(device=device).manual_seed(args.seed * 1000 + k)
        U = torch.randn(args.I, args.R, dtype=torch.float64, device=device, generator=g)
        u = torch.rand(args.I, dtype=torch.float64, device=device, generator=g)
        w = torch.pow(1.0 - torch.rand(args.I, dtype=torch.float64, device=device, generator=g), -1.0 / 1.5)
        U *= torch.where(u < 0.01, w, torch.ones_like(w))[:, None]
        fs.append(U)
    return fs


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled by NVML every ~2 ms from a thread while
    the timed region runs (the recipe's clocks line; nvidia-smi -lms is too coarse
    for a region of a few tens of ms)."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.err = None
        self._stop = threading.Event()
        self.t = None

    def _sample(self):
        import pynvml
        sm = pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        try:
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.samples.append((sm, r))

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(0.002)

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._sample()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as ex:
            self.err = str(ex)

    def stop(self):
        if self.t is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"nvml unavailable: {self.err}"]}
        self._stop.set()
        self.t.join()
        import statistics
        sm = [x for x, _ in self.samples]
        reasons = sorted({nm for _, r in self.samples for bit, nm in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.smax, "reasons": reasons,
                "samples": len(sm)}


# ---------------------------------------------------------------- roofline
def descent_bytes(idx, dims, R, excluded=None, elt=8):
    """Algorithmic (compulsory) HBM bytes of one step's draw kernels:
    per included factor, every distinct stored Gram the walks read (root + left
    child of every internal node on a drawn path) x P x 8, every distinct leaf's
    rows x R x elt, the E-tree (R stored packed Grams) and V, plus the per-draw
    state traffic (h read+write, index write)."""
    import numpy as np
    P = R * (R + 1) // 2
    J = idx.shape[0]
    total = 0
    per_pos = []
    inc = [k for k in range(len(dims)) if excluded is None or k != excluded]
    for pos, k in enumerate(inc):
        I = dims[k]
        L = (I + R - 1) // R
        d = int(np.ceil(np.log2(L))) if L > 1 else 0
        bottom = 2 * L - (1 << d)
        leaves = np.unique(idx[:, k].astype(np.int64) // R)
        node = np.where(leaves < bottom, (1 << d) - 1 + leaves, L - 1 + (leaves - bottom))
        internal = set()
        v = node.copy()
        while True:
            v = v[v > 0]
            if v.size == 0:
                break
            v = np.unique((v - 1) // 2)
            internal.update(v.tolist())
        grams = 1 + len(internal)  # root + one left child per internal node on a path
        rows_read = sum(min(R, I - int(l) * R) for l in leaves)
        b = grams * P * 8 + rows_read * R * elt
        b += R * P * 8 + R * R * 8  # E-tree + eigenvectors
        b += J * R * 8 * (2 if pos > 0 else 1) + J * 4  # h in/out, index
        per_pos.append(b)
        total += b
    return total, per_pos


DMMA_PEAK_TFLOPS = 37.0  # measured FP64 tensor (DMMA) peak on this pool's B200 (profiles/r01_fp64_peak_probe.txt)


def one_stage_flops(idx, dims, R, excluded=None):
    """Algorithmic FP64 flops of one one-stage step (north_star M = G+ o hh^T o G_{>k}):
    per draw and included factor, one packed quadratic form R(R+1) per internal node on
    its root-to-leaf path plus the normaliser, and per leaf row scanned up to the pick
    (the reference's early exit, segment_tree_sampler.cpp:284-291) R (r o h) + R(R+1)."""
    import numpy as np
    total = 0
    inc = [k for k in range(len(dims)) if excluded is None or k != excluded]
    qf = R * (R + 1)
    for k in inc:
        I = dims[k]
        L = (I + R - 1) // R
        d = int(np.ceil(np.log2(L))) if L > 1 else 0
        bottom = 2 * L - (1 << d)
        t = idx[:, k].astype(np.int64)
        leaf = t // R
        depth = np.where(leaf < bottom, d, d - 1)
        scanned = t - leaf * R + 1
        total += int(((depth + 1) * qf).sum()) + int((scanned * (qf + R)).sum())
    return total


# ---------------------------------------------------------------- reference arm
def cpu_reference_run(host_factors, J, seed, steps, warmup, keep=None, one_stage=False):
    """The reference's own CPU sampler (oracle/_ref: unmodified sources), all host cores.
    Returns (construction s, per-step seconds, reference handle if keep, last outputs)."""
    import oracle
    if not oracle.ref_available():
        raise RuntimeError("oracle/_ref not built")
    t0 = time.perf_counter()
    s = oracle.OracleKrp(host_factors, "ref")
    build_s = time.perf_counter() - t0
    for i in range(warmup):
        s.sample(None, J, seed + 100 + i, one_stage=one_stage)
    times = []
    out = None
    for i in range(steps):
        t0 = time.perf_counter()
        out = s.sample(None, J, seed + i, one_stage=one_stage)
        times.append(time.perf_counter() - t0)
    return build_s, times, (s if keep else None), out


def parity_against_reference(ref, ours, last_seed, J, N, one_stage=False):
    """Compare the timed call (and the exclude-one calls) with the reference's own
    KrpSampler::sample on the same factors and seeds (krp_sampler.cpp:82-151).
    `ours[e]` = (idx, prob, rows, margin, seed) host arrays of our call for exclusion e."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from parity_util import BOUNDARY_TOL, compare_draws, rel_err_vec, rows_rel_err
    tot = {"against": "reference KrpSampler::sample (oracle/_ref), same factors and seeds, every draw",
           "calls": [], "checked": 0, "mismatches": 0, "boundary_draws": 0, "unexplained": 0,
           "max_prob_rel_err": 0.0, "max_rows_rel_err": 0.0, "boundary_tol": BOUNDARY_TOL}
    for e, (gi, gp, gr, gm, sd, first) in ours.items():
        if first is not None:
            ri, rp, rr = first
        else:
            ri, rp, rr = ref.sample(None if e == "none" else int(e), J, sd, one_stage=one_stage)
        n, nb, nu = compare_draws(gi, gm, ri)
        same = ~np.any(gi != ri, axis=1)
        pe = rel_err_vec(gp[same], rp[same])
        re_ = rows_rel_err(gr[same], rr[same])
        tot["calls"].append({"excluded": e, "seed": sd, "draws": int(J), "mismatches": n, "boundary": nb,
                             "unexplained": nu, "prob_rel_err": pe, "rows_rel_err": re_})
        tot["checked"] += int(J)
        tot["mismatches"] += n
        tot["boundary_draws"] += nb
        tot["unexplained"] += nu
        tot["max_prob_rel_err"] = max(tot["max_prob_rel_err"], pe)
        tot["max_rows_rel_err"] = max(tot["max_rows_rel_err"], re_)
    tot["ok"] = tot["unexplained"] == 0 and tot["max_prob_rel_err"] <= 1e-10
    return tot


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch
    dev = "cuda:0" if torch.cuda.is_available() else "cpu"
    fs = [f.cpu().numpy() for f in make_factors(args, dev)]
    torch.cuda.empty_cache() if torch.cuda.is_available() else None
    cores = os.cpu_count()
    build_s, times, _, _ = cpu_reference_run(fs, args.J, args.seed, args.steps, args.warmup,
                                             one_stage=args.mode == "one_stage")
    tot = sum(times)
    value = args.J * len(times) / tot
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": bench_config(args, world),
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": "reference",
                         "sample": f"full step: KrpSampler::sample(nullopt, J={args.J}) on config 2 "
                                   f"(OMP threads={os.environ.get('OMP_NUM_THREADS', cores)}); "
                                   f"construction {build_s:.1f} s untimed",
                         "compile": REF_FLAGS},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "build_s": build_s,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")

    from paper_2301_12584_b200 import KrpSampler

    fs = make_factors(args, dev)
    torch.cuda.synchronize()
    s = KrpSampler.from_device(fs, device=local)
    if args.tune:
        s.set_tuning(**{k: int(v) for k, v in (t.split("=", 1) for t in args.tune)})
    R, N, J = args.R, args.N, args.J
    dims = [args.I] * N

    # ---- tree build timing (device events, replicated on each rank) ----
    s.profile_enable(True)
    s.profile_read(reset=True)
    for j in range(N):
        s.rebuild(j)
    pb = s.profile_read(reset=True)
    build_ms = (pb["tree_leaf"]["ms"] + pb["tree_levels"]["ms"]) / N
    P = R * (R + 1) // 2
    L = (args.I + R - 1) // R
    build_bytes = args.I * R * 8 + L * P * 8
    peak, peak_kind = load_peaks()

    idx = torch.empty(J, N, dtype=torch.int32, device=dev)
    prob = torch.empty(J, dtype=torch.float64, device=dev)
    rows = torch.empty(J, R, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.ExternalStream(s.stream(), device=dev)

    def step(i, excluded=None):
        s.sample_device(excluded, J, args.seed + i, idx, prob, rows, mode=args.mode, draw_offset=rank * J)

    # Steps are issued asynchronously (KRPG_OPT_ASYNC): each call returns once its
    # kernels are enqueued, so its host setup (the R x R eigensolves) overlaps the
    # previous call's kernels. Every call still does all of its work; errors are
    # collected by s.sync() at the end of the region.
    s.set_async(True)
    for i in range(args.warmup):
        step(10_000 + i)
    s.sync()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    s.profile_read(reset=True)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(float(i))  # L2 flush (256 MiB write) before every step, inside the region
        step(i)
    e1.record(stream)
    s.sync()
    torch.cuda.synchronize()
    clk = clocks.stop()
    s.set_async(False)
    if world > 1:
        dist.barrier()
    prof = s.profile_read(reset=True)
    elapsed_ms = e0.elapsed_time(e1)
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    value = world * J * args.steps / (elapsed_ms / 1e3)
    launches = sum(v["launches"] for v in prof.values())

    # ---- roofline of the dominant kernel (draws) from this run's own paths ----
    idx_h = idx.cpu().numpy().view(np.uint32)
    bytes_step, _ = descent_bytes(idx_h, dims, R)
    flops_step = one_stage_flops(idx_h, dims, R) if args.mode == "one_stage" else None
    draws_ms = prof["draws"]["ms"] / args.steps
    achieved = bytes_step / (draws_ms / 1e3) / 1e9
    share = prof["draws"]["ms"] / max(elapsed_ms, 1e-9)
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get("draws_bytes_per_step")
        except Exception:
            traffic = None

    # profiling events only inside the timed region above (kernel time for the roofline);
    # the rest measures the API as a user calls it
    s.profile_enable(False)

    # ---- the timed call's outputs (last step), and a deterministic re-run with margins ----
    last_seed = args.seed + args.steps - 1
    ours = {}

    def keep(e, seed_, excluded):
        mg = torch.empty(J, dtype=torch.float64, device=dev)
        i2, p2, r2 = torch.empty_like(idx), torch.empty_like(prob), torch.empty_like(rows)
        s.sample_device(excluded, J, seed_, i2, p2, r2, mg, mode=args.mode, draw_offset=rank * J)
        s.sync()
        det = bool(torch.equal(i2, idx) and torch.equal(p2, prob) and torch.equal(r2, rows))
        ours[e] = (idx.cpu().numpy().view(np.uint32), prob.cpu().numpy(), rows.cpu().numpy(),
                   mg.cpu().numpy(), seed_, None)
        return det

    deterministic = keep("none", last_seed, None)

    # ---- exclude-one rates (device-timed, not part of the headline) ----
    excl = {}
    for k in range(N):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        step(500 + k, excluded=k)
        e1.record(stream)
        torch.cuda.synchronize()
        excl[str(k)] = J / (e0.elapsed_time(e1) / 1e3)
        deterministic &= keep(str(k), args.seed + 500 + k, k)

    # ---- e2e: the public host API (host outputs, copies inside the region) ----
    e2e_t = []
    b = None
    for i in range(3):  # untimed: the pinned output buffers of two live batches are cached
        b = s.sample(None, J, args.seed + 700 + i, mode=args.mode, draw_offset=rank * J)
    for i in range(args.e2e_steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        b = s.sample(None, J, args.seed + 777 + i, mode=args.mode, draw_offset=rank * J)
        e2e_t.append(time.perf_counter() - t0)
    tt = torch.tensor([sum(e2e_t)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e_value = world * J * len(e2e_t) / float(tt.item())
    h2d = 8 * (P + N * (R * R + R))  # per-call operand upload (G+, eigenvectors, eigenvalues)
    d2h = J * (N * 4 + 8 + R * 8)   # indices, probabilities, rows

    # ---- multi-GPU construction, N > 1 only ----
    construction = None
    if world > 1:
        try:
            construction = time_construction(s, fs, args, dist, torch, dev)
        except Exception as ex:  # reported, never hides the headline
            construction = {"error": f"{type(ex).__name__}: {ex}"}

    # ---- cpu_baseline leg: the reference on the same factors; parity of the timed call ----
    cpu_base = None
    parity = {"deterministic_rerun": deterministic}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            host = [f.cpu().numpy() for f in fs]
            build_s, times, ref, out = cpu_reference_run(host, J, last_seed, steps=1, warmup=0, keep=True,
                                                         one_stage=args.mode == "one_stage")
            cpu_base = {"value": J / times[0], "unit": "samples/s", "cores": os.cpu_count(),
                        "kind": "reference", "compile": REF_FLAGS,
                        "sample": f"one KrpSampler::sample(nullopt, J={J}) of the reference on the same "
                                  f"config-2 factors, all host cores (construction {build_s:.1f} s untimed)"}
            gi, gp, gr, gm, sd, _ = ours["none"]
            ours["none"] = (gi, gp, gr, gm, sd, out)
            parity.update(parity_against_reference(ref, ours, last_seed, J, N, one_stage=args.mode == "one_stage"))
            del ref
        except Exception as ex:  # reported, never silently substituted
            cpu_base = {"value": None, "unit": "samples/s", "cores": os.cpu_count(), "kind": "reference",
                        "sample": f"unavailable: {type(ex).__name__}: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(args, world),
            "issue": "asynchronous calls (KRPG_OPT_ASYNC): host setup overlaps the previous step's kernels",
            "tuning": dict(t.split("=", 1) for t in args.tune) or "defaults",
            "roofline": ({"bound": "hbm", "kernel": "k_draws (batched root-to-leaf descent)",
                          "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                          "traffic": traffic, "peak_kind": peak_kind,
                          "alg_bytes_per_step": bytes_step, "kernel_ms_per_step": draws_ms,
                          "kernel_share_of_step": share} if args.mode == "two_stage" else
                         {"bound": "tensor", "kernel": "one-stage descent (k_eval_reg with B = G_v o Y, k_leaf_os)",
                          "achieved": flops_step / (draws_ms / 1e3) / 1e12, "peak": DMMA_PEAK_TFLOPS,
                          "unit": "TFLOP/s", "frac": flops_step / (draws_ms / 1e3) / 1e12 / DMMA_PEAK_TFLOPS,
                          "traffic": None, "peak_kind": "measured FP64 DMMA (profiles/r01_fp64_peak_probe.txt)",
                          "alg_flops_per_step": flops_step, "kernel_ms_per_step": draws_ms,
                          "kernel_share_of_step": share, "hbm_alg_bytes_per_step": bytes_step}),
            "cpu_baseline": cpu_base,
            "parity": parity,
            "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clk,
            "tree_build": {"ms_per_factor": build_ms, "alg_bytes_per_factor": build_bytes,
                           "achieved_gbs": build_bytes / (build_ms / 1e3) / 1e9,
                           "frac": build_bytes / (build_ms / 1e3) / 1e9 / peak,
                           "flops_per_factor": args.I * R * (R + 1)},
            "exclude_one_samples_per_s": excl,
            "kernel_ms_per_step": {k: v["ms"] / args.steps for k, v in prof.items() if v["launches"]},
        }
        if construction is not None:
            line["construction"] = construction
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def time_construction(s, fs, args, dist, torch, dev):
    """N > 1: rebuild factor 0 three ways, device-timed, max over ranks.
    (a) row-partitioned: each rank builds the subtree of its rows, the level slices
        and subtree roots are all-gathered over NCCL, the top levels reduced locally;
    (b) (a) plus the all-gather of the factor's row slices (what a row-partitioned
        producer, e.g. the STS-CP solve, has to add so every rank can scan leaves);
    (c) all-gather U's row slices + redundant full rebuild on every rank.
    (a) is checked bit-identical to the single-GPU build."""
    from paper_2301_12584_b200.sharding import build_partitioned
    world, rank = dist.get_world_size(), dist.get_rank()
    I, R = args.I, args.R
    U = fs[0]
    ref_tree = s.tree_device(0).clone()
    rows = (I + world - 1) // world
    mine = torch.zeros(rows * args.R, dtype=U.dtype, device=dev)
    lo, hi = rank * rows, min(I, (rank + 1) * rows)
    mine[:(hi - lo) * R] = U[lo:hi].reshape(-1)
    gathered = torch.empty(world * rows * R, dtype=U.dtype, device=dev)

    def timed(fn, reps=3):
        best = None
        for _ in range(reps):
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            best = float(dt.item()) if best is None else min(best, float(dt.item()))
        return best * 1e3

    def ag_u():
        dist.all_gather_into_tensor(gathered, mine)

    ms_a = timed(lambda: build_partitioned(s, 0))
    same = bool(torch.equal(s.tree_device(0), ref_tree))
    ms_b = timed(lambda: (ag_u(), build_partitioned(s, 0)))
    ms_c = timed(lambda: (ag_u(), s.rebuild(0)))
    ms_u = timed(ag_u)
    return {"factor": 0, "ranks": world, "partitioned_ms": ms_a, "partitioned_plus_allgather_U_ms": ms_b,
            "allgather_U_plus_rebuild_ms": ms_c, "allgather_U_ms": ms_u,
            "partitioned_bit_identical_to_single_build": same,
            "timing": "host wall clock around device-synchronised calls, best of 3, max over ranks"}


def respawn_under_torchrun(args):
    """`python bench.py --gpus N` (N > 1) without torchrun: re-execute under
    torch.distributed.run, one process per GPU, rendezvous on 127.0.0.1."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execvpe(sys.executable, cmd, env)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        respawn_under_torchrun(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
