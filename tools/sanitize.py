#!/usr/bin/env python
"""Small workloads that touch every device kernel family, for compute-sanitizer.

    compute-sanitizer --tool racecheck python tools/sanitize.py [case ...]

Cases (all small so the instrumented run finishes in minutes):
  sample    config-2-shaped two-stage draws (R = 64, deep trees so the shallow
            level kernel, the first-position tables and the fused deep pass all
            run), with and without an exclusion, plus the unfused path
  onestage  one-stage (general-Y) draws and the exact conditional
  rank      R = 128 / 256 (split and streamed level kernels, R > 64 leaf scan)
  update    batched single-entry updates and a whole-factor rebuild
  sts       sparse-tensor ingestion and one STS-CP solve
  prodlev   CP-ARLS-LEV product sampler
Each case asserts against the device's own invariants only (no oracle), so the
sanitizer report is the result.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2301_12584_b200 as pkg  # noqa: E402


def factors(shapes, seed):
    rng = np.random.default_rng(seed)
    out = []
    for I, R in shapes:
        U = rng.standard_normal((I, R))
        w = (1.0 - rng.random(I)) ** (-1.0 / 1.5)
        out.append(U * np.where(rng.random(I) < 0.01, w, 1.0)[:, None])
    return out


def case_sample():
    fs = factors([(1 << 16, 64), (40000, 64), (3 << 13, 64)], 1)
    s = pkg.KrpSampler(fs)
    for e in (None, 1):
        b = s.sample(e, 4096, 7, margin=True)
        assert np.all(np.isfinite(b.probabilities)) and np.all(b.probabilities > 0)
    s.set_fused_deep(False)
    b2 = s.sample(None, 4096, 7)
    s.set_fused_deep(True)
    b1 = s.sample(None, 4096, 7)
    assert b1.indices.shape == b2.indices.shape  # both paths ran (they may differ at rounding level)
    b3 = s.sample(0, 50000, 8, margin=True)  # many shallow levels with many runs per warp
    assert np.all(b3.probabilities > 0)
    s.close()


def case_onestage():
    fs = factors([(3000, 16), (2049, 16), (4096, 16)], 2)
    s = pkg.KrpSampler(fs)
    b = s.sample(None, 2048, 9, mode="one_stage")
    assert np.all(b.probabilities > 0)
    cd = s.conditional(None, 1, np.ones(16))
    assert abs(cd.probabilities.sum() - 1.0) < 1e-9
    s.close()
    fs = factors([(40000, 64), (30000, 64)], 12)  # grouped one-stage, several levels
    s = pkg.KrpSampler(fs)
    assert np.all(s.sample(0, 8192, 3, mode="one_stage").probabilities > 0)
    s.close()
    fs = factors([(20000, 128), (3000, 128)], 13)  # R = 128: split level kernel + split leaf
    s = pkg.KrpSampler(fs)
    assert np.all(s.sample(None, 4096, 4, mode="one_stage").probabilities > 0)
    s.close()


def case_rank():
    for R in (128, 256):
        fs = factors([(R * 300, R), (R * 129, R)], 3)
        s = pkg.KrpSampler(fs)
        b = s.sample(None, 1024, 11)
        assert np.all(b.probabilities > 0)
        s.close()


def case_update():
    fs = factors([(20000, 32), (7000, 32), (9000, 32)], 4)
    s = pkg.KrpSampler(fs)
    rng = np.random.default_rng(5)
    n = 2000
    s.update_factor_entries(1, rng.integers(0, 7000, n), rng.integers(0, 32, n), rng.standard_normal(n))
    s.update_factor(2, factors([(9500, 32)], 6)[0])
    b = s.sample(None, 2048, 3)
    assert np.all(b.probabilities > 0)
    s.close()


def case_sts():
    rng = np.random.default_rng(7)
    dims = [3000, 2000, 1500]
    nnz = 60000
    coords = np.stack([np.minimum(rng.zipf(1.1, nnz) - 1, d - 1) for d in dims], axis=1).astype(np.uint32)
    vals = rng.lognormal(0.0, 1.0, nnz)
    T = pkg.SparseTensor(dims, coords, vals)
    fs = factors([(d, 16) for d in dims], 8)
    s = pkg.KrpSampler(fs)
    for j in range(3):
        sg = s.sts_solve(T, j, 4096, 100 + j)
        assert np.all(np.isfinite(sg))
    s.close()
    T.close()


def case_prodlev():
    fs = factors([(5000, 64), (3000, 64), (4000, 64)], 9)
    s = pkg.KrpSampler(fs)
    b = s.product_lev_sample(None, 4096, 1)
    assert np.all(b.probabilities > 0)
    s.close()


CASES = {"sample": case_sample, "onestage": case_onestage, "rank": case_rank, "update": case_update,
         "sts": case_sts, "prodlev": case_prodlev}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        CASES[nm]()
        print(f"sanitize case {nm}: ok", flush=True)
