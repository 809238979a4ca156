import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    # make sure the checker and the product library exist (nvcc/gcc cross-build, no GPU needed)
    port = os.path.join(ROOT, "oracle", "build", "libkrp_oracle.so")
    if not os.path.exists(port):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True,
                       stdout=subprocess.DEVNULL)
    lib = os.path.join(ROOT, "paper_2301_12584_b200", "lib", "libkrpg.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2301_12584_b200", "csrc"), "-j8"],
                       check=True, stdout=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def have_ref():
    import oracle
    return oracle.ref_available()
