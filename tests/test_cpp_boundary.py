"""The drop-in boundary compiled from C++: tests/cpp/facade_test.cpp drives the
engine through include/mpcr_b200_mpnum.hpp with the reference's own host types
(mpnum::MPArray, GemmParams, the exception hierarchy) and compares every call
with the reference CPU library on the same inputs, including the
NotPositiveDefinite rethrow that chol_with_jitter (workloads.cpp:54-70)
catches.  The binary is built in this container (tests/cpp/Makefile, called
by __graft_entry__.build()) and travels to the GPU box."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "facade_test")
REF_INC = "/root/reference/proj/core/include"


def test_facade_header_compiles():
    """The façade and the C header compile as C++20 against the reference headers."""
    if not os.path.isdir(REF_INC):
        pytest.skip("reference headers absent (GPU box)")
    src = '#include "mpcr_b200_mpnum.hpp"\nint main() { return 0; }\n'
    out = subprocess.run(["g++", "-std=gnu++20", "-fsyntax-only", "-Wall", "-Werror", "-I",
                          os.path.join(ROOT, "include"), "-I", REF_INC, "-x", "c++", "-"],
                         input=src, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr[-3000:]


@pytest.mark.gpu
def test_facade_vs_reference_on_gpu():
    if not os.path.exists(BIN):
        pytest.fail(f"{BIN} missing: run __graft_entry__.build() where /root/reference exists")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0 and "facade ok" in out.stdout, out.stdout[-3000:] + out.stderr[-2000:]
