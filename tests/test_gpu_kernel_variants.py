"""The descent's alternative kernel paths compute bit-identical draws.

The level kernel k_eval_reg (register-resident Gram, pre-doubled off-diagonal
fragments) and the first-position tables (E-tree and top factor-tree levels
computed once per (node, eigen-component) when h = ones) are claimed to apply
exactly the arithmetic of the per-draw DMMA quadratic form (block_qf_packed) to
exactly the same operands, so every branch decision, probability, row and
margin must equal the k_eval_cta path bit for bit -- and so must other deep /
shallow splits and deep-pass work-unit sizes, and the multi-level cooperative launch
(k_eval_reg_ml: grid barriers instead of kernel boundaries). The variants are per-handle
options (krpg_set_option, KRPG_OPT_EVAL_REG ...), switched on one sampler.
"""
import numpy as np
import pytest

from parity_util import pareto_factors

pytestmark = pytest.mark.gpu


def draws(s, n_factors, J):
    out = {}
    for ex in (None, 0, n_factors - 1):
        b = s.sample(ex, J, seed=777, margin=True)
        key = "none" if ex is None else str(ex)
        out["idx_" + key] = b.indices.copy()
        out["prob_" + key] = b.probabilities.copy()
        out["rows_" + key] = b.rows.copy()
        out["margin_" + key] = b.margin.copy()
    return out


def same(a, b, what):
    for k, v in a.items():
        assert np.array_equal(b[k], v), f"{what}: {k} differs"


@pytest.mark.parametrize("shapes,J", [
    ([(1 << 16, 64), (40000, 64), (50000, 64)], 32768),   # level kernel + deep pass + first-position tables
    ([(20000, 32), (30000, 32), (9000, 32)], 20000),      # R = 32, J not a multiple of the warp ranges
    ([(5000, 24), (3000, 24)], 4096),                     # non-power-of-two E-tree (parked leaves)
    ([(70000, 64), (3000, 64)], 200000),                  # J beyond one resident wave: the multi-level launch falls back to one launch per level
])
def test_level_kernel_and_tables_bit_identical(shapes, J):
    from paper_2301_12584_b200 import KrpSampler
    s = KrpSampler(pareto_factors(shapes, seed=11, frac=0.01))
    # block_qf_packed order: the CTA kernel, the register-resident kernel, the tables
    s.set_tuning(eval_split=0, eval_reg=0, pos0_tables=0)
    base = draws(s, len(shapes), J)
    for opts in ({"eval_reg": 1, "pos0_tables": 0}, {"eval_reg": 0, "pos0_tables": 1},
                 {"eval_reg": 1, "pos0_tables": 1}, {"deep_threshold": 64}, {"deep_threshold": 16},
                 {"deep_chunk": 32}, {"deep_chunk": 3}, {"deep_chunk": 0},
                 # one launch per level instead of the multi-level cooperative launch, and back
                 {"eval_ml": 0}, {"eval_ml": 0, "pos0_tables": 0}, {"eval_ml": 1}, {"pos0_tables": 1}):
        s.set_tuning(**opts)
        same(base, draws(s, len(shapes), J), opts)
    # split order (R = 64: the Gram split over a CTA's warps): the split kernel on every
    # level vs the first-position tables computed in the same order
    s.set_tuning(eval_reg=1, pos0_tables=0, deep_threshold=32, deep_chunk=8, eval_split=1)
    base = draws(s, len(shapes), J)
    s.set_tuning(pos0_tables=1)
    same(base, draws(s, len(shapes), J), "split order with tables")
    s.set_tuning(eval_split=16)
    s.close()


def test_one_stage_multi_level_launch_bit_identical():
    """One-stage mode (B = G_v o Y): the multi-level cooperative launch against one launch per level."""
    from paper_2301_12584_b200 import KrpSampler
    s = KrpSampler(pareto_factors([(30000, 32), (9000, 32), (20000, 32)], seed=5, frac=0.01))
    out = []
    for ml in (0, 1):
        s.set_tuning(eval_ml=ml)
        b = s.sample(1, 20000, seed=99, mode="one_stage", margin=True)
        out.append((b.indices.copy(), b.probabilities.copy(), b.rows.copy(), b.margin.copy()))
    for x, y in zip(*out):
        assert np.array_equal(x, y)
    s.close()


def test_tuning_option_errors():
    from paper_2301_12584_b200 import KrpgInvalidArgument, KrpSampler
    s = KrpSampler(pareto_factors([(300, 8), (200, 8)], seed=1))
    with pytest.raises(KrpgInvalidArgument):
        s.set_tuning(deep_chunk=33)
    with pytest.raises(KrpgInvalidArgument):
        s.set_tuning(eval_split=2)
    with pytest.raises(KrpgInvalidArgument):
        s.set_tuning(nonsense=1)
    s.close()
