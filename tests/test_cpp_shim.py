"""The C++ host mirror (include/cpstream_b200.hpp) compiles and links against
the C-ABI library on CPU; on the GPU its restatement of the reference's
proj/tests/test_streaming.cpp runs through the B200 kernels."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_streaming_b200.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "_build", "test_streaming_b200")


@pytest.fixture(scope="module")
def binary():
    from paper_1807_01350_b200 import build
    lib = build.build(verbose=False)
    libdir = os.path.dirname(lib)
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-Wall", "-I" + os.path.join(ROOT, "include"),
                           "-I" + os.path.join(ROOT, "paper_1807_01350_b200", "csrc"), SRC,
                           "-L" + libdir, "-locten_b200", "-Wl,-rpath," + libdir, "-o", OUT])
    return OUT


def test_cpp_shim_builds_and_links(binary):
    assert os.access(binary, os.X_OK)
    # every symbol resolves at load time (ldd-style check without running compute)
    out = subprocess.run(["ldd", binary], capture_output=True, text=True).stdout
    assert "libocten_b200.so" in out and "not found" not in out.split("libocten_b200.so")[1].split("\n")[0]


@pytest.mark.gpu
def test_cpp_shim_reference_streaming_cases(binary):
    r = subprocess.run([binary], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
