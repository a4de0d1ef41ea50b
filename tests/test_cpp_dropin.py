"""The drop-in C++ API (include/neuzip/*.hpp, same names and signatures as
/root/reference/proj/include/neuzip) compiles against the C ABI with the
reference's own toolchain flags, and -- on a B200 -- passes the
acceptance-style suite in tests/cpp/dropin_test.cpp."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
BIN = os.path.join(ROOT, "build", "dropin_test")
LIBDIR = os.path.join(ROOT, "paper_2410_20650_b200")


def build_dropin() -> str:
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-pthread", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           SRC, "-L", LIBDIR, "-lnzgpu", f"-Wl,-rpath,{LIBDIR}", "-o", BIN]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return BIN


def test_dropin_headers_compile_and_link():
    assert os.path.exists(build_dropin())


def test_dropin_headers_are_self_contained():
    for h in ("errors", "bitfloat", "ans", "tensorstore", "parallel", "neuzip"):
        src = f'#include "neuzip/{h}.hpp"\nint main() {{ return 0; }}\n'
        out = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Werror", "-I",
                              os.path.join(ROOT, "include"), "-x", "c++", "-"], input=src, capture_output=True,
                             text=True)
        assert out.returncode == 0, (h, out.stderr)


@pytest.mark.gpu
def test_dropin_acceptance_suite_on_gpu():
    binary = build_dropin()
    out = subprocess.run([binary], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failed" in out.stdout
