"""The reference's OWN unit tests (test_krp_sampler.cpp, test_segment_tree.cpp,
test_rng.cpp, test_sketch.cpp), compiled unmodified against the B200 drop-in headers and libkrpg.so
(oracle/Makefile target `_ref/refsuite`, built where /root/reference exists), run
on the device -- all cases, the five sparse-construction ones (from_sparse over
variable leaf segments) included."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "refsuite")
SKIP = ""


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="reference test suite not built (needs /root/reference)")
def test_reference_unit_tests_pass_on_the_device_drop_in():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900, env={**os.environ, "REFSUITE_SKIP": SKIP})
    print(r.stdout[-3000:])
    summary = [ln for ln in r.stdout.splitlines() if ln.startswith("refsuite:")]
    assert summary, r.stdout + r.stderr
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert " 0 failed," in summary[0]
