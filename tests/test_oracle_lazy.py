"""CPU: the lazy full-size restatement (oracle/lazy.py) against the C oracle (pinned to
the reference) on enumerable problems: indices equal up to counted boundary draws,
probabilities and rows within 1e-10 relative on matching draws."""
import numpy as np
import pytest

import oracle
from oracle.lazy import LazyKrp, Topology
from parity_util import compare_draws, pareto_factors, rel_err_vec, rows_rel_err


@pytest.mark.parametrize("shapes,seed", [([(500, 8), (300, 8), (257, 8)], 1), ([(2000, 16), (999, 16)], 2),
                                         ([(1000, 12), (700, 12), (64, 12)], 3)])
def test_lazy_restatement_matches_oracle(shapes, seed):
    fs = pareto_factors(shapes, seed)
    o = oracle.OracleKrp(fs, "port")
    lz = LazyKrp(fs)
    draws = np.arange(0, 400) + 1000
    for e in [None] + list(range(len(shapes))):
        ri, rp, rr, rm = o.sample(e, 400, 77, want_margin=True, draw_offset=1000)
        li, lp, lr, lm = lz.sample(e, draws, 77)
        n, nb, nu = compare_draws(li, lm, ri, rm)
        assert nu == 0
        same = ~np.any(li != ri, axis=1)
        assert rel_err_vec(lp[same], rp[same]) <= 1e-10
        assert rows_rel_err(lr[same], rr[same]) <= 1e-12


def test_lazy_topology_matches_reference_segments():
    for I, F in [(4096, 16), (777, 24), (1000, 8), (130, 5), (64, 4), (1, 3)]:
        t = Topology(I, F)
        ot = oracle.OracleTree(np.ones((I, 2)), F, None, "port")
        assert t.n == ot.node_count and t.L == ot.leaf_count
        for v in range(t.n):
            assert t.rows(v) == ot.node_segment(v)
