"""Tree-build time per factor (config 2: 2^22 x 64 fp64), rebuilds checked bit-identical
to the first build. (Round 2 also timed forced-occupancy leaf-kernel variants here:
profiles/r02_tree_variants.jsonl; they lost and were removed.)"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from bench import load_peaks, make_factors  # noqa: E402
from paper_2301_12584_b200 import KrpSampler  # noqa: E402


class A:
    N, I, R, seed = 1, 1 << 22, 64, 2301


fs = make_factors(A(), "cuda")
s = KrpSampler.from_device(fs)
ref = s.tree_device(0).clone()
peak, _ = load_peaks()
P = 64 * 65 // 2
alg = A.I * 64 * 8 + (A.I // 64) * P * 8
for v in (0,):
    s.profile_enable(True)
    s.rebuild(0)
    s.profile_read(reset=True)
    for _ in range(5):
        s.rebuild(0)
    pb = s.profile_read(reset=True)
    ms = (pb["tree_leaf"]["ms"] + pb["tree_levels"]["ms"]) / 5
    same = bool(torch.equal(s.tree_device(0), ref))
    print(json.dumps({"leaf_variant": v, "ms_per_factor": ms, "leaf_ms": pb["tree_leaf"]["ms"] / 5,
                      "levels_ms": pb["tree_levels"]["ms"] / 5, "levels_launches": pb["tree_levels"]["launches"] / 5,
                      "achieved_gbs": alg / (ms / 1e3) / 1e9, "frac": alg / (ms / 1e3) / 1e9 / peak,
                      "bit_identical": same}), flush=True)
