"""Generate the golden fixtures from the reference itself (oracle/_ref, the
unmodified /root/reference sources compiled by oracle/Makefile).

    python tests/golden/make_golden.py

Writes tests/golden/golden_v1.npz. The fixtures pin the oracle restatement
(tests/test_oracle.py, CPU) and the device sampler (tests/test_gpu_parity.py).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
from parity_util import config1_factors, digest, spiked_factors  # noqa: E402


def main():
    assert oracle.ref_available(), "build oracle/_ref first (make -C oracle)"
    ref = oracle.backend("ref")
    out = {}
    # rng.hpp known answers
    out["rng_u_42_3"] = ref.uniforms(42, 3, 64)
    out["rng_n_11_0"] = ref.normals(11, 0, 64)
    out["derive_seed"] = np.array([ref.derive_seed(1, 2, 3), ref.derive_seed(1, 3, 2),
                                   ref.derive_seed(2301, 1, 0)], dtype=np.uint64)

    # config 1: 3 x 4096 x 16, Pareto rows, J = 8192
    fs = config1_factors(kind="ref")
    out["c1_digest"] = np.array(digest(fs))
    s = oracle.OracleKrp(fs, "ref")
    J, seed = 8192, 12584
    out["c1_J"] = np.array(J)
    out["c1_seed"] = np.array(seed)
    for e in (None, 0, 1, 2):
        idx, prob, rows = s.sample(e, J, seed)
        tag = "none" if e is None else str(e)
        out[f"c1_idx_{tag}"] = idx
        out[f"c1_prob_{tag}"] = prob
        out[f"c1_rowsum_{tag}"] = rows.sum(axis=1)
    idx, prob, rows = s.sample(None, J, seed, one_stage=True)
    out["c1_idx_one_stage"] = idx
    out["c1_prob_one_stage"] = prob
    for j in range(3):
        out[f"c1_gram_{j}"] = s.factor_gram(j)
    out["c1_node_ids"] = np.array([0, 1, 3, 5, 7, 63, 127, 255, 509], dtype=np.uint64)
    out["c1_nodes_f0"] = np.stack([s.node_gram(0, int(v)) for v in out["c1_node_ids"]])

    # Figure-5 fixture: spiked 8x8x3 (support.hpp:21-31), exact leverage + draws
    sp = spiked_factors([(8, 8)] * 3, 620, kind="ref")
    out["sp_digest"] = np.array(digest(sp))
    out["sp_leverage"] = ref.leverage(sp)
    ss = oracle.OracleKrp(sp, "ref")
    idx, prob, _ = ss.sample(None, 4096, 621)
    out["sp_idx"] = idx
    out["sp_prob"] = prob
    h = np.array([0.3, -1.2, 0.8, 0.1, 2.0, -0.5, 0.7, 1.1])
    p, m = ss.conditional(None, 1, h)
    out["sp_cond_h"] = h
    out["sp_cond_p"] = p
    out["sp_cond_mix"] = m

    # dense kernels
    B = ref.normals(7, 0, 32 * 16).reshape(32, 16)
    G = B.T @ B
    V, lam = ref.eigh(G)
    out["eig_G"] = G
    out["eig_lam"] = lam
    out["eig_absV"] = np.abs(V)
    P, rk = ref.pinv(G)
    out["pinv"] = P
    out["pinv_rank"] = np.array(rk)

    # updates: 20 random single-entry updates on a 2-factor sampler
    fu = [oracle.random_matrix(10, 3, 760 + j, kind="ref") for j in range(2)]
    su = oracle.OracleKrp(fu, "ref")
    rr = np.array([4, 1, 9, 4, 0, 7, 4, 2], dtype=np.uint64)
    cc = np.array([1, 0, 2, 1, 2, 0, 0, 1], dtype=np.uint32)
    vv = ref.normals(762, 0, rr.size)
    su.update_entries(0, rr, cc, vv)
    out["upd_r"], out["upd_c"], out["upd_v"] = rr, cc, vv
    out["upd_gram0"] = su.factor_gram(0)
    idx, prob, _ = su.sample(None, 400, 763)
    out["upd_idx"] = idx

    path = os.path.join(HERE, "golden_v1.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
