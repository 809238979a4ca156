"""The C++ drop-in (include/krplev/*.hpp over libkrpg.so): compiles anywhere
(CPU test), and its parity program runs on the GPU (gpu test)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
LIBDIR = os.path.join(ROOT, "paper_2301_12584_b200", "lib")
ORACLE = os.path.join(ROOT, "oracle")


def build(tmp_path):
    exe = str(tmp_path / "test_dropin")
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", f"-I{ROOT}/include", f"-I{ORACLE}",
           SRC, "-o", exe, f"-L{LIBDIR}", "-lkrpg", f"-L{ORACLE}/build", "-lkrp_oracle",
           f"-Wl,-rpath,{LIBDIR}", f"-Wl,-rpath,{ORACLE}/build", "-Wl,-rpath,/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_dropin_headers_compile_and_link(tmp_path):
    build(tmp_path)


@pytest.mark.gpu
def test_cpp_dropin_parity(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
