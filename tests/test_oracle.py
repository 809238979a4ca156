"""CPU: pin the oracle restatement (oracle/krp_oracle.c) against the reference.

1. bit-for-bit against the committed golden fixtures (generated from the
   reference itself by tests/golden/make_golden.py) — runs everywhere;
2. bit-for-bit against oracle/_ref (the unmodified reference sources compiled
   here) on fresh random cases — runs where oracle/_ref was built;
3. the reference's own known-answer tests (test_krp_sampler.cpp,
   test_segment_tree.cpp) restated on the oracle.
"""
import os
from functools import lru_cache

import numpy as np
import pytest

import oracle
from parity_util import config1_factors, digest, spiked_factors

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz")


@lru_cache(maxsize=1)
def golden():
    return dict(np.load(GOLDEN))


# ---------------------------------------------------------------- golden pins
def test_rng_golden():
    g = golden()
    port = oracle.backend("port")
    assert np.array_equal(port.uniforms(42, 3, 64), g["rng_u_42_3"])
    assert np.array_equal(port.normals(11, 0, 64), g["rng_n_11_0"])
    assert [port.derive_seed(1, 2, 3), port.derive_seed(1, 3, 2), port.derive_seed(2301, 1, 0)] == \
        [int(x) for x in g["derive_seed"]]


def test_config1_golden_two_stage_and_one_stage():
    g = golden()
    fs = config1_factors()
    assert digest(fs) == str(g["c1_digest"])
    s = oracle.OracleKrp(fs, "port")
    J, seed = int(g["c1_J"]), int(g["c1_seed"])
    for e in (None, 0, 1, 2):
        tag = "none" if e is None else str(e)
        idx, prob, rows = s.sample(e, J, seed)
        assert np.array_equal(idx, g[f"c1_idx_{tag}"]), tag
        assert np.array_equal(prob, g[f"c1_prob_{tag}"]), tag
        assert np.array_equal(rows.sum(axis=1), g[f"c1_rowsum_{tag}"]), tag
    idx, prob, _ = s.sample(None, J, seed, one_stage=True)
    assert np.array_equal(idx, g["c1_idx_one_stage"])
    assert np.array_equal(prob, g["c1_prob_one_stage"])
    for j in range(3):
        assert np.array_equal(s.factor_gram(j), g[f"c1_gram_{j}"])
    for v, G in zip(g["c1_node_ids"], g["c1_nodes_f0"]):
        assert np.array_equal(s.node_gram(0, int(v)), G)


def test_spiked_golden():
    g = golden()
    sp = spiked_factors([(8, 8)] * 3, 620)
    assert digest(sp) == str(g["sp_digest"])
    port = oracle.backend("port")
    assert np.array_equal(port.leverage(sp), g["sp_leverage"])
    s = oracle.OracleKrp(sp, "port")
    idx, prob, _ = s.sample(None, 4096, 621)
    assert np.array_equal(idx, g["sp_idx"])
    assert np.array_equal(prob, g["sp_prob"])
    p, m = s.conditional(None, 1, g["sp_cond_h"])
    assert np.array_equal(p, g["sp_cond_p"])
    assert np.array_equal(m, g["sp_cond_mix"])


def test_dense_golden():
    g = golden()
    port = oracle.backend("port")
    V, lam = port.eigh(g["eig_G"])
    assert np.array_equal(lam, g["eig_lam"])
    assert np.array_equal(np.abs(V), g["eig_absV"])
    P, rk = port.pinv(g["eig_G"])
    assert np.array_equal(P, g["pinv"])
    assert rk == int(g["pinv_rank"])


def test_updates_golden():
    g = golden()
    fu = [oracle.random_matrix(10, 3, 760 + j) for j in range(2)]
    s = oracle.OracleKrp(fu, "port")
    s.update_entries(0, g["upd_r"], g["upd_c"], g["upd_v"])
    assert np.array_equal(s.factor_gram(0), g["upd_gram0"])
    idx, _, _ = s.sample(None, 400, 763)
    assert np.array_equal(idx, g["upd_idx"])


# ------------------------------------------------- live reference comparison
ref_only = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built here")

CASES = [
    ([(8, 3), (7, 3), (6, 3)], 11),
    ([(64, 4), (40, 4), (33, 4)], 12),
    ([(300, 8), (257, 8), (100, 8)], 13),
    ([(129, 5), (77, 5)], 14),
    ([(1000, 16), (1, 16), (513, 16)], 15),
]


@ref_only
@pytest.mark.parametrize("shapes,seed", CASES)
def test_port_matches_reference_bitwise(shapes, seed):
    fs = [oracle.random_matrix(r, c, seed * 10 + k) for k, (r, c) in enumerate(shapes)]
    a = oracle.OracleKrp(fs, "port")
    b = oracle.OracleKrp(fs, "ref")
    for j in range(len(fs)):
        assert np.array_equal(a.factor_gram(j), b.factor_gram(j))
    for e in [None] + list(range(len(fs))):
        for one in (False, True):
            ia, pa, ra = a.sample(e, 1500, seed, one_stage=one)
            ib, pb, rb = b.sample(e, 1500, seed, one_stage=one)
            assert np.array_equal(ia, ib) and np.array_equal(pa, pb) and np.array_equal(ra, rb)
    h = oracle.random_matrix(1, shapes[0][1], seed)[0]
    for k in range(len(fs)):
        pa, ma = a.conditional(None, k, h)
        pb, mb = b.conditional(None, k, h)
        assert np.array_equal(pa, pb) and np.array_equal(ma, mb)
    r = np.array([0, 1, 0, shapes[0][0] - 1], dtype=np.uint64)
    c = np.array([0, 1, 1, 0], dtype=np.uint32)
    v = np.array([0.5, -1.0, 2.0, 3.0])
    a.update_entries(0, r, c, v)
    b.update_entries(0, r, c, v)
    assert np.array_equal(a.factor_gram(0), b.factor_gram(0))
    n_nodes = 2 * ((shapes[0][0] + shapes[0][1] - 1) // shapes[0][1]) - 1
    for node in [0] + list(range(1, n_nodes, 2)):
        assert np.array_equal(a.node_gram(0, node), b.node_gram(0, node))
    assert np.array_equal(a.sample(None, 500, 9)[0], b.sample(None, 500, 9)[0])


@ref_only
def test_port_tree_matches_reference_full_layout():
    for I, R, F in [(64, 4, 4), (29, 3, 3), (33, 3, 4), (1, 2, 2), (100, 6, 7)]:
        U = oracle.random_matrix(I, R, 400 + I)
        Y = oracle.random_matrix(2 * R, R, 500 + I)
        Y = Y.T @ Y
        for y in (None, Y):
            a = oracle.OracleTree(U, F, y, "port")
            b = oracle.OracleTree(U, F, y, "ref", full=True)
            assert a.node_count == b.node_count and a.leaf_count == b.leaf_count
            for v in range(a.node_count):
                assert a.node_segment(v) == b.node_segment(v)
                assert np.array_equal(a.node_gram(v), b.node_gram(v))
            h = oracle.random_matrix(1, R, 7)[0]
            assert np.array_equal(a.row_sample(h, 5, 2, 300), b.row_sample(h, 5, 2, 300))


def sparse_coo(I, R, density, seed):
    rng = np.random.default_rng(seed)
    U = np.where(rng.random((I, R)) < density, rng.standard_normal((I, R)), 0.0)
    U[0, 0] = 1.5
    r, c = np.nonzero(U)  # row-major order
    return U, r, c, U[r, c]


@ref_only
@pytest.mark.parametrize("I,R,density", [(64, 4, 0.1), (200, 3, 0.3), (500, 5, 0.6), (40, 6, 1.0), (6, 3, 0.0)])
def test_port_sparse_tree_matches_reference(I, R, density):
    """from_sparse (segment_tree_sampler.cpp:67-109): the port's greedy partition over
    densified rows gives the reference's leaves, Grams (bitwise) and draws."""
    U, r, c, v = sparse_coo(I, R, density, I + R)
    a = oracle.OracleTree.from_sparse(I, R, r, c, v, "port")
    b = oracle.OracleTree.from_sparse(I, R, r, c, v, "ref", full=True)
    assert a.node_count == b.node_count and a.leaf_count == b.leaf_count
    for node in range(a.node_count):
        assert a.node_segment(node) == b.node_segment(node)
        assert np.array_equal(a.node_gram(node), b.node_gram(node))
    for lf in range(a.leaf_count):
        f, l = int(a.offsets[lf]), int(a.offsets[lf + 1])
        assert (np.count_nonzero(U[f:l]) <= R * R) or (l - f == 1)
    h = oracle.random_matrix(1, R, 8)[0]
    assert np.array_equal(a.row_sample(h, 5, 2, 300), b.row_sample(h, 5, 2, 300))


@ref_only
@pytest.mark.parametrize("excluded", [None, 0, 2])
def test_port_product_lev_matches_reference(excluded):
    """CP-ARLS-LEV product_lev_sample (sketch.cpp:86-149): the port's restatement is
    bitwise the reference's (indices, probabilities, rows)."""
    fs = [oracle.random_matrix(n, 6, 700 + n) for n in (40, 90, 17)]
    fs[1][::7] *= 10.0
    a = oracle.backend("port").product_lev_sample(fs, excluded, 3000, 31)
    b = oracle.backend("ref").product_lev_sample(fs, excluded, 3000, 31)
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(x, y)


@ref_only
def test_port_eigh_matches_reference():
    port, ref = oracle.backend("port"), oracle.backend("ref")
    for n in (1, 2, 5, 16, 33):
        B = oracle.random_matrix(2 * n, n, 900 + n)
        G = B.T @ B
        Vp, lp = port.eigh(G)
        Vr, lr = ref.eigh(G)
        assert np.array_equal(lp, lr) and np.array_equal(Vp, Vr)


# ------------------------------------- reference known answers on the oracle
def normalized_leverage(fs):
    return oracle.backend("port").leverage(fs)


def chained_joint(s, shapes, excluded):
    """test_krp_sampler.cpp:23-51: chain the exact conditionals."""
    inc = [k for k in range(len(shapes)) if excluded is None or k != excluded]
    R = shapes[0][1]
    total = int(np.prod([shapes[k][0] for k in inc]))
    joint = np.zeros(total)

    def walk(pos, h, prefix, flat):
        if pos == len(inc):
            joint[flat] = prefix
            return
        k = inc[pos]
        p, _ = s.conditional(excluded, k, h)
        for t in range(p.size):
            if p[t] <= 0.0:
                continue
            walk(pos + 1, h * s.factors[k][t], prefix * p[t], flat * shapes[k][0] + t)

    walk(0, np.ones(R), 1.0, 0)
    return joint


@pytest.mark.parametrize("shapes,excluded", [
    ([(6, 2), (5, 2)], None),
    ([(8, 3), (7, 3), (6, 3)], None),
    ([(4, 4), (16, 4), (9, 4)], 1),
    ([(12, 2), (3, 2), (10, 2)], 2),
])
def test_oracle_joint_exactness(shapes, excluded):
    """test_krp_sampler.cpp:126-153: chained conditionals == normalized leverage (1e-8)."""
    fs = [oracle.random_matrix(r, c, 701 + k) for k, (r, c) in enumerate(shapes)]
    s = oracle.OracleKrp(fs, "port")
    joint = chained_joint(s, shapes, excluded)
    inc = [fs[k] for k in range(len(fs)) if excluded is None or k != excluded]
    q = normalized_leverage(inc)
    assert np.max(np.abs(joint - q)) <= 1e-8


def test_oracle_identity_and_uniform_known_answers():
    # test_krp_sampler.cpp:82-107
    s = oracle.OracleKrp([np.ones((2, 1)), np.ones((2, 1))], "port")
    idx, prob, _ = s.sample(None, 40000, 610)
    flat = idx[:, 0] * 2 + idx[:, 1]
    counts = np.bincount(flat, minlength=4)
    chi2 = np.sum((counts - 10000.0) ** 2 / 10000.0)
    assert chi2 < 11.345
    assert np.allclose(prob, 0.25)
    s = oracle.OracleKrp([np.eye(2), np.eye(2)], "port")
    idx, _, _ = s.sample(None, 100000, 611)
    flat = idx[:, 0] * 2 + idx[:, 1]
    counts = np.bincount(flat, minlength=4)
    assert counts[1] == 0 and counts[2] == 0


def test_oracle_errors():
    with pytest.raises(oracle.OracleInvalidArgument):
        oracle.OracleKrp([np.zeros((2, 2)), np.zeros((2, 2))], "port")
    s = oracle.OracleKrp([np.ones((3, 2)), np.ones((4, 2))], "port")
    with pytest.raises(oracle.OracleInvalidArgument):
        s.sample(5, 10, 1)
    with pytest.raises(oracle.OracleInvalidArgument):
        s.sample(None, 0, 1)
