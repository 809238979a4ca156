"""Device SegmentTreeSampler (krpg_segtree_*) against the reference's
SegmentTreeSampler through the oracle (test_segment_tree.cpp's checks on device):
node Grams, batched row_sample bit-exact up to counted boundary draws, analytic
probabilities = enumerated q_{h,U,Y}, update_entry, errors."""
import numpy as np
import pytest

import oracle
from parity_util import pareto_factors, rel_err_matrix

pytestmark = pytest.mark.gpu
TOL = 1e-10


def ST():
    from paper_2301_12584_b200 import SegmentTreeSampler
    return SegmentTreeSampler


def exact_q(U, h, Y):
    X = U * h[None, :]
    m = np.einsum("ia,ab,ib->i", X, Y, X)
    return m / m.sum()


def psd(R, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((R + 3, R))
    return A.T @ A / R


SHAPES = [(1000, 16, 16), (777, 8, 5), (513, 24, 1), (2049, 32, 64), (300, 12, 7), (64, 4, 64)]


@pytest.mark.parametrize("I,R,F", SHAPES)
@pytest.mark.parametrize("kind", ["ones", "general"])
def test_segtree_matches_reference_tree(I, R, F, kind):
    U = pareto_factors([(I, R)], seed=I + R + F)[0]
    Y = psd(R, I) if kind == "general" else None
    t = ST()(U, F, Y=Y, y=None if Y is not None else np.ones(R))
    o = oracle.OracleTree(U, F, Y, "port")
    L, n = t.shape()
    assert (L, n) == (o.leaf_count, o.node_count)
    for v in [0] + list(range(1, n, 2)):
        assert rel_err_matrix(t.node_gram(v), o.node_gram(v)) <= TOL
    rng = np.random.default_rng(7)
    J = 400
    H = rng.standard_normal((J, R))
    got, mg = t.row_sample_batch(H, seed=11, stream0=100, counter=1, margin=True)
    ref = np.array([o.row_sample(H[d], 11, 100 + d, 1)[0] for d in range(J)])
    bad = got != ref
    assert np.all(mg[bad] <= TOL), f"{int(bad.sum())} mismatches outside the boundary margin"
    q = t.analytic_probabilities(H[0])
    assert np.max(np.abs(q - exact_q(U, H[0], Y if Y is not None else np.ones((R, R))))) <= 1e-10


def test_segtree_rank1_vector_y_and_counters():
    """Rank-1 y (the reference's fold z = h o y path) vs the general Y = y y^T tree
    (same distribution), and successive counters of one CounterRng stream."""
    I, R, F = 1500, 16, 16
    U = pareto_factors([(I, R)], seed=3)[0]
    y = np.linspace(0.5, 1.5, R)
    t = ST()(U, F, y=y)
    o = oracle.OracleTree(U, F, np.outer(y, y), "port")
    rng = np.random.default_rng(1)
    h = rng.standard_normal(R)
    seq = o.row_sample(h, 5, 9, 50)  # counters 1..50 of CounterRng(5, 9)
    for c in range(1, 51):
        got, mg = t.row_sample_batch(h[None, :], 5, 9, counter=c, margin=True)
        assert got[0] == seq[c - 1] or mg[0] <= TOL
    q = t.analytic_probabilities(h)
    assert np.max(np.abs(q - exact_q(U, h, np.outer(y, y)))) <= 1e-10


def test_segtree_update_entry_matches_rebuild():
    I, R, F = 900, 8, 8
    U = pareto_factors([(I, R)], seed=4)[0]
    t = ST()(U, F, y=np.ones(R))
    rng = np.random.default_rng(2)
    for _ in range(40):
        r, c, v = int(rng.integers(I)), int(rng.integers(R)), float(rng.standard_normal())
        t.update_entry(r, c, v)
        U[r, c] = v
    o = oracle.OracleTree(U, F, None, "port")
    for v in [0] + list(range(1, o.node_count, 2)):
        assert rel_err_matrix(t.node_gram(v), o.node_gram(v)) <= 1e-9


def test_segtree_errors():
    from paper_2301_12584_b200 import KrpgError, KrpgInvalidArgument
    U = np.ones((10, 4))
    with pytest.raises(KrpgInvalidArgument):
        ST()(U, 0, y=np.ones(4))
    with pytest.raises(KrpgInvalidArgument):
        ST()(U, 2, Y=np.eye(4), y=np.ones(4))
    t = ST()(U, 2, y=np.ones(4))
    with pytest.raises(KrpgInvalidArgument):
        t.node_gram(2)  # right child: not stored in the compact layout
    with pytest.raises(KrpgError):
        t.row_sample_batch(np.zeros((1, 4)), 1)  # C = 0: degenerate distribution


def sparse_coo(I, R, density, seed):
    rng = np.random.default_rng(seed)
    U = np.where(rng.random((I, R)) < density, rng.standard_normal((I, R)), 0.0)
    U[0, 0] = 1.5
    r, c = np.nonzero(U)
    return U, r, c, U[r, c]


SPARSE = [(64, 4, 0.1), (200, 3, 0.3), (6, 3, 0.0), (3000, 16, 0.05), (20000, 32, 0.1), (5000, 24, 0.9),
          (1537, 8, 0.02)]


@pytest.mark.parametrize("I,R,density", SPARSE)
def test_segtree_from_sparse_matches_reference(I, R, density):
    """from_sparse (segment_tree_sampler.cpp:67-109): device tree over the greedy
    R^2-nonzero leaf segments vs the oracle's; draws vs the oracle and vs the dense
    device tree over the same rows (partition-independent inverse CDF)."""
    U, r, c, v = sparse_coo(I, R, density, I * R)
    t = ST().from_sparse(I, R, r, c, v)
    o = oracle.OracleTree.from_sparse(I, R, r, c, v, "port")
    assert t.sparse()
    assert np.array_equal(t.leaf_offsets(), o.offsets)
    L, n = t.shape()
    assert (L, n) == (o.leaf_count, o.node_count)
    for node in range(n):
        assert t.node_segment(node) == o.node_segment(node)
    for node in [0] + list(range(1, n, 2)):
        assert rel_err_matrix(t.node_gram(node), o.node_gram(node)) <= TOL
    rng = np.random.default_rng(I)
    J = 300
    H = rng.standard_normal((J, R))
    got, mg = t.row_sample_batch(H, seed=21, stream0=7, counter=1, margin=True)
    ref = np.array([o.row_sample(H[d], 21, 7 + d, 1)[0] for d in range(J)])
    bad = got != ref
    assert np.all(mg[bad] <= TOL), f"{int(bad.sum())} mismatches outside the boundary margin"
    dense = ST()(U, R, y=np.ones(R))
    got2, mg2 = dense.row_sample_batch(H, seed=21, stream0=7, counter=1, margin=True)
    bad2 = got2 != got
    assert np.all(np.minimum(mg, mg2)[bad2] <= TOL)
    q = t.analytic_probabilities(H[0])
    assert np.max(np.abs(q - exact_q(U, H[0], np.ones((R, R))))) <= 1e-10


def test_segtree_from_sparse_update_and_errors():
    from paper_2301_12584_b200 import KrpgInvalidArgument
    I, R = 400, 4
    U, r, c, v = sparse_coo(I, R, 0.3, 5)
    t = ST().from_sparse(I, R, r, c, v)
    rng = np.random.default_rng(3)
    for k in rng.choice(len(v), 30, replace=False):
        val = float(rng.standard_normal())
        t.update_entry(int(r[k]), int(c[k]), val)
        U[r[k], c[k]] = val
    zr, zc = np.argwhere(U == 0.0)[0]
    with pytest.raises(KrpgInvalidArgument):
        t.update_entry(int(zr), int(zc), 1.0)  # outside the stored pattern
    rr, cc = np.nonzero(U)
    o = oracle.OracleTree.from_sparse(I, R, rr, cc, U[rr, cc], "port")
    if np.array_equal(o.offsets, t.leaf_offsets()):  # same pattern -> same partition
        for node in [0] + list(range(1, o.node_count, 2)):
            assert rel_err_matrix(t.node_gram(node), o.node_gram(node)) <= 1e-9
    with pytest.raises(KrpgInvalidArgument):
        ST().from_sparse(3, 2, [1, 0], [0, 0], [1.0, 2.0])  # unsorted
    with pytest.raises(KrpgInvalidArgument):
        ST().from_sparse(3, 2, [], [], [])  # no nonzeros
