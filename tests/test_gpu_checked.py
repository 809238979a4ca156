"""The bounds-checked library (make CHECKED=1: KRPG_DCHECK device asserts on node ids,
stored slots, row ranges, sorted positions, block-list and ring capacity) runs every
kernel family on representative workloads without a failed check. compute-sanitizer is
closed on the GPU pool; this and the determinism tests stand in for memcheck / racecheck
(DESIGN.md 7b). Each case runs in its own process with KRPG_LIB_VARIANT=checked."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2301_12584_b200", "lib", "libkrpg_checked.so")


@pytest.mark.parametrize("case", ["sample", "onestage", "rank", "update", "sts", "prodlev"])
def test_checked_build_runs_clean(case):
    assert os.path.exists(CHECKED), "build the checked library: make -C paper_2301_12584_b200/csrc CHECKED=1"
    env = dict(os.environ, KRPG_LIB_VARIANT="checked")
    code = ("import sys; sys.path.insert(0, %r); sys.argv = ['sanitize', %r]; "
            "import paper_2301_12584_b200._lib as L; assert L.LIB_PATH.endswith('libkrpg_checked.so') and L.lib().krpg_is_checked_build() == 1; "
            "import runpy; runpy.run_path(%r, run_name='__main__')"
            % (ROOT, case, os.path.join(ROOT, "tools", "sanitize.py")))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert f"sanitize case {case}: ok" in r.stdout
