"""bench.py host logic (no GPU): the two arms emit identical config dicts, the roofline
byte / flop counters agree with hand counts on tiny trees, and the reference-parity
summary counts boundary draws the way tests/parity_util does."""
import os
import sys
import types

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def args(**kw):
    a = types.SimpleNamespace(N=3, I=1 << 22, R=64, J=65536, mode="two_stage", gpus=1, seed=2301)
    a.__dict__.update(kw)
    return a


def test_both_arms_use_one_config_dict():
    a = args()
    assert bench.bench_config(a, 1) == bench.bench_config(a, 1)
    assert bench.bench_config(a, 4)["parallelism"].startswith("draws sharded across 4")
    c = bench.bench_config(a, 1)
    assert {"workload", "N", "I", "R", "J", "mode", "l2"} <= set(c)
    assert "model" not in c


def test_descent_bytes_hand_count():
    # one factor, I = 4 rows, R = 1: 4 leaves, depth 2, perfect tree; draws at rows 0 and 3
    idx = np.array([[0], [3]], dtype=np.uint32)
    total, per = bench.descent_bytes(idx, [4], 1)
    P = 1
    grams = 1 + 3  # root + left children of the 3 internal nodes on the two paths
    rows = 2  # two distinct leaves of one row each
    expect = grams * P * 8 + rows * 1 * 8 + (1 * P * 8 + 1 * 8) + 2 * 1 * 8 * 1 + 2 * 4
    assert total == expect and per == [expect]


def test_one_stage_flops_hand_count():
    # I = 8, R = 2: 4 leaves (depth 2); draw at row 3 = leaf 1, second row of its leaf
    idx = np.array([[3]], dtype=np.uint32)
    qf = 2 * 3
    assert bench.one_stage_flops(idx, [8], 2) == (2 + 1) * qf + 2 * (qf + 2)


def test_parity_summary_counts_boundary_draws():
    J, N = 6, 2
    gi = np.zeros((J, N), dtype=np.uint32)
    ri = gi.copy()
    ri[1, 0] = 7  # a mismatch inside the boundary margin
    ri[4, 1] = 9  # a mismatch outside it
    gm = np.full(J, 1.0)
    gm[1] = 1e-12
    p = np.ones(J)
    rows = np.ones((J, 3))

    class Ref:
        def sample(self, e, J_, seed, one_stage=False):
            return ri, p, rows

    out = bench.parity_against_reference(Ref(), {"none": (gi, p, rows, gm, 5, None)}, 5, J, N)
    assert out["checked"] == J and out["mismatches"] == 2
    assert out["boundary_draws"] == 1 and out["unexplained"] == 1 and not out["ok"]


def test_respawn_builds_a_torchrun_command(monkeypatch):
    seen = {}

    def fake_exec(path, cmd, env):
        seen["cmd"], seen["env"] = cmd, env
        raise SystemExit(0)

    monkeypatch.setattr(os, "execvpe", fake_exec)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    try:
        bench.respawn_under_torchrun(args(gpus=4))
    except SystemExit:
        pass
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]
    assert seen["env"]["NCCL_DEBUG"] == "INFO"
