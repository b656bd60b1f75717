"""The header-only C++ wrapper (include/embc_b200.hpp) compiles against the C
ABI (CPU), and its test program passes on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2407_04272_b200")
SRC = os.path.join(ROOT, "tests", "cpp", "api_test.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "api_test")


def _build():
    from paper_2407_04272_b200 import _lib
    _lib.lib()
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(cuda, "include"), SRC,
           "-o", BIN, "-L", PKG, "-lembc_cuda", f"-Wl,-rpath,{PKG}", "-L", os.path.join(cuda, "lib64"), "-lcudart",
           f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_cpp_wrapper_compiles():
    _build()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_cpp_wrapper_runs():
    _build()
    r = subprocess.run([BIN, ROOT], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "api_test: ok" in r.stdout
