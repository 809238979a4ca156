"""The descent's alternative kernel paths compute bit-identical draws.

The level kernel k_eval_reg (register-resident Gram, pre-doubled off-diagonal
fragments) and the first-position tables (E-tree and top factor-tree levels
computed once per (node, eigen-component) when h = ones) are claimed to apply
exactly the arithmetic of the per-draw DMMA quadratic form (block_qf_packed) to
exactly the same operands, so every branch decision, probability, row and
margin must equal the k_eval_cta path bit for bit. The variants are selected by
environment switches that are read once per process, so each runs in its own
subprocess on the same factors and seeds.
"""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, sys.argv[1] + "/tests")
from parity_util import pareto_factors
from paper_2301_12584_b200 import KrpSampler
shapes = [(int(a), int(b)) for a, b in (x.split("x") for x in sys.argv[3].split(","))]
fs = pareto_factors(shapes, seed=int(sys.argv[4]), frac=0.01)
s = KrpSampler(fs)
out = {}
for ex in (None, 0, len(shapes) - 1):
    b = s.sample(ex, int(sys.argv[5]), seed=777, margin=True)
    key = "none" if ex is None else str(ex)
    out["idx_" + key] = b.indices
    out["prob_" + key] = b.probabilities
    out["rows_" + key] = b.rows
    out["margin_" + key] = b.margin
np.savez(sys.argv[2], **out)
"""


def run_variant(env_extra, shapes, seed, J):
    fd, path = tempfile.mkstemp(suffix=".npz")
    os.close(fd)
    env = dict(os.environ)
    env.update(env_extra)
    spec = ",".join(f"{i}x{r}" for i, r in shapes)
    subprocess.run([sys.executable, "-c", CHILD, ROOT, path, spec, str(seed), str(J)], env=env, check=True,
                   timeout=600)
    d = dict(np.load(path))
    os.unlink(path)
    return d


@pytest.mark.parametrize("shapes,J", [
    ([(1 << 16, 64), (40000, 64), (50000, 64)], 32768),   # level kernel + deep pass + first-position tables
    ([(20000, 32), (30000, 32), (9000, 32)], 20000),      # R = 32, J not a multiple of the warp ranges
    ([(5000, 24), (3000, 24)], 4096),                     # non-power-of-two E-tree (parked leaves)
])
def test_level_kernel_and_tables_bit_identical(shapes, J):
    # block_qf_packed order: the CTA kernel, the register-resident kernel, the tables
    base = run_variant({"KRPG_EVAL_SPLIT": "0", "KRPG_EVAL_REG": "0", "KRPG_POS0_TABLES": "0"}, shapes, 11, J)
    for extra in ({"KRPG_EVAL_SPLIT": "0", "KRPG_EVAL_REG": "1", "KRPG_POS0_TABLES": "0"},
                  {"KRPG_EVAL_SPLIT": "0", "KRPG_EVAL_REG": "0", "KRPG_POS0_TABLES": "1"},
                  {"KRPG_EVAL_SPLIT": "0"}):
        got = run_variant(extra, shapes, 11, J)
        for k, v in base.items():
            assert np.array_equal(got[k], v), f"{extra}: {k} differs"
    # split order (R = 64: the Gram split over a CTA's warps): the split kernel on every
    # level vs the first-position tables computed in the same order
    base = run_variant({"KRPG_EVAL_SPLIT": "1", "KRPG_POS0_TABLES": "0"}, shapes, 11, J)
    got = run_variant({"KRPG_EVAL_SPLIT": "1"}, shapes, 11, J)
    for k, v in base.items():
        assert np.array_equal(got[k], v), f"split order with tables: {k} differs"
