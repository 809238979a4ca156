"""Device CP-ARLS-LEV product sampler (krpg_product_lev_sample[_factors],
sketch.cpp:86-149) against the oracle's restatement (pinned
bitwise to the reference's product_lev_sample in tests/test_oracle.py):

  * per-row leverage scores u_i^T pinv(G) u_i (DMMA kernel for R % 8 == 0 up to
    160, the generic kernel otherwise; fp64 and fp32 storage) vs numpy, 1e-10;
  * indices bit-exact up to counted boundary draws (|cum - target| <= 1e-10,
    normalised), probabilities 1e-10 relative, rows bit-exact where indices agree;
  * the per-mode distribution against the product of exact leverage scores (chi-square);
  * the reference's errors."""
import numpy as np
import pytest

import oracle
from parity_util import compare_draws, pareto_factors, rel_err_vec

pytestmark = pytest.mark.gpu
TOL = 1e-10


def lib():
    import paper_2301_12584_b200 as p
    return p


def exact_lev(U):
    G = U.T @ U
    w, V = np.linalg.eigh(G)
    keep = w > len(w) * np.finfo(float).eps * w.max()
    Gp = (V[:, keep] / w[keep]) @ V[:, keep].T
    return np.einsum("ia,ab,ib->i", U, Gp, U)


def exact_lev_sumsq(U):
    """normalised leverage as sums of squares in the eigenbasis (no cancellation)"""
    w, V = np.linalg.eigh(U.T @ U)
    keep = w > len(w) * np.finfo(float).eps * w.max()
    p = ((U @ (V[:, keep] / np.sqrt(w[keep]))) ** 2).sum(1)
    return p / p.sum()


def cond(U):
    w = np.linalg.eigvalsh(U.T @ U)
    return float(w.max() / w[w > len(w) * np.finfo(float).eps * w.max()].min())


@pytest.mark.parametrize("R", [8, 16, 24, 32, 40, 64, 80, 96, 128, 160, 5, 72, 192, 256])
@pytest.mark.parametrize("fp32", [False, True])
def test_leverage_scores_match_numpy(R, fp32):
    I = 3001 if R <= 64 else 1501
    U = pareto_factors([(I, R), (64, R)], seed=R)
    s = lib().KrpSampler(U, storage="f32" if fp32 else "f64")
    Ud = s.factor(0)  # what the device stores (fp32-rounded when fp32)
    got = s.leverage_scores(0)
    ref = exact_lev(Ud)
    assert np.max(np.abs(got - ref)) <= 1e-10 * max(1.0, np.max(np.abs(ref)))
    assert abs(got.sum() - R) <= 1e-8 * R  # leverage scores sum to the rank


SHAPES = [
    [(4096, 16)] * 3,
    [(1000, 8), (777, 8), (1500, 8)],
    [(3000, 64), (2048, 64), (513, 64)],
    [(900, 72), (700, 72)],          # generic kernel
    [(2000, 128), (1000, 128)],
    [(50, 4), (70, 4), (33, 4), (20, 4)],
]


@pytest.mark.parametrize("shapes", SHAPES)
@pytest.mark.parametrize("excluded", [None, 0, 1])
def test_product_lev_matches_oracle(shapes, excluded):
    fs = pareto_factors(shapes, seed=sum(i for i, _ in shapes))
    J = 20000
    s = lib().KrpSampler(fs)
    b = s.product_lev_sample(excluded, J, seed=77, margin=True)
    o_idx, o_prob, o_rows, o_mg = oracle.backend("port").product_lev_sample(fs, excluded, J, 77)
    n, nb, bad = compare_draws(b.indices, b.margin, o_idx, o_mg, TOL)
    assert bad == 0, f"{bad} of {n} mismatching draws outside the boundary margin"
    ok = np.all(b.indices == o_idx, axis=1)
    # probabilities: 1e-10 against exactly computed leverage; against the reference
    # also the error of its pseudo-inverse -- cyclic Jacobi stops at off-norm <=
    # 1e-12 |G|_F (dense_kernels.cpp:93-176), i.e. ~1e-12 cond(G_k) per factor
    inc = [k for k in range(len(fs)) if k != excluded]
    exact = [exact_lev_sumsq(fs[k]) for k in inc]
    pex = np.prod([exact[q][b.indices[:, k].astype(np.int64)] for q, k in enumerate(inc)], axis=0)
    assert rel_err_vec(b.probabilities, pex) <= TOL
    tol_ref = TOL + 1e-12 * sum(cond(fs[k]) for k in inc)
    assert rel_err_vec(b.probabilities[ok], o_prob[ok]) <= tol_ref
    assert np.array_equal(b.rows[ok], o_rows[ok])
    if excluded is not None:
        assert np.all(b.indices[:, excluded] == 0xFFFFFFFF)
    # the free function (factors from the host, gram(U) on the device) draws the same
    f = lib().product_lev_sample(fs, excluded, J, 77, margin=True)
    n2, nb2, bad2 = compare_draws(f.indices, f.margin, o_idx, o_mg, TOL)
    assert bad2 == 0
    assert np.array_equal(f.indices[ok & np.all(f.indices == b.indices, axis=1)],
                          b.indices[ok & np.all(f.indices == b.indices, axis=1)])


def test_product_lev_draw_offset_and_fp32():
    fs = pareto_factors([(2000, 32)] * 3, seed=5)
    s = lib().KrpSampler(fs)
    a = s.product_lev_sample(None, 4000, seed=3)
    b = s.product_lev_sample(None, 1000, seed=3, draw_offset=3000)
    assert np.array_equal(a.indices[3000:], b.indices)  # streams keyed by the global draw id
    s32 = lib().KrpSampler(fs, storage="f32")
    c = s32.product_lev_sample(None, 4000, seed=3, margin=True)
    o = oracle.backend("port").product_lev_sample([s32.factor(k) for k in range(3)], None, 4000, 3)
    assert compare_draws(c.indices, c.margin, o[0], o[3], TOL)[2] == 0


def test_product_lev_distribution_chi_square():
    """Per draw the joint law is the product of the per-mode normalised leverage
    scores (sketch.cpp:86-149); pooled Pearson chi-square at alpha = 0.001."""
    fs = pareto_factors([(16, 4), (12, 4), (10, 4)], seed=11)
    ps = [exact_lev(U) / exact_lev(U).sum() for U in fs]
    joint = np.einsum("i,j,k->ijk", *ps).ravel()
    J = 1 << 21
    s = lib().KrpSampler(fs)
    b = s.product_lev_sample(None, J, seed=1234)
    flat = (b.indices[:, 0].astype(np.int64) * 12 + b.indices[:, 1]) * 10 + b.indices[:, 2]
    counts = np.bincount(flat, minlength=joint.size)
    exp = joint * J
    keep = exp >= 5
    chi2 = float(np.sum((counts[keep] - exp[keep]) ** 2 / exp[keep]))
    dof = int(keep.sum()) - 1
    from scipy.stats import chi2 as chi2d
    assert chi2 < chi2d.ppf(0.999, dof), (chi2, dof)
    # reported probability = product of the per-mode probabilities
    assert rel_err_vec(b.probabilities[:1000], joint[flat[:1000]]) <= 1e-10


def test_product_lev_errors():
    from paper_2301_12584_b200 import KrpgError, KrpgInvalidArgument
    fs = pareto_factors([(100, 8)] * 2, seed=1)
    s = lib().KrpSampler(fs)
    with pytest.raises(KrpgInvalidArgument):
        s.product_lev_sample(None, 0, 1)
    with pytest.raises(KrpgInvalidArgument):
        s.product_lev_sample(2, 10, 1)
    with pytest.raises(KrpgInvalidArgument):
        lib().product_lev_sample([fs[0]], 0, 10, 1)  # no factors left
    with pytest.raises(KrpgInvalidArgument):
        lib().product_lev_sample([], None, 10, 1)
    with pytest.raises(KrpgError):
        lib().product_lev_sample([fs[0], np.zeros((5, 8))], None, 10, 1)  # zero factor


def test_product_lev_large_factors():
    """2^20 x 64 factors: tables over a million rows, leverage sums = rank, draws vs
    the oracle on the same inputs (indices up to boundary draws)."""
    fs = pareto_factors([(1 << 20, 64)] * 3, seed=9, frac=0.01)
    s = lib().KrpSampler(fs)
    for k in range(3):
        assert abs(s.leverage_scores(k).sum() - 64) <= 1e-7 * 64
    J = 65536
    b = s.product_lev_sample(None, J, seed=5, margin=True)
    o = oracle.backend("port").product_lev_sample(fs, None, J, 5)
    assert compare_draws(b.indices, b.margin, o[0], o[3], TOL)[2] == 0
