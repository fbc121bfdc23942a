"""The C++ drop-in header (include/hgks_b200/hgks.hpp) driven the way the
reference's own doctest suites drive hgks:: (tests/native/test_dropin.cpp):
residual/face-count/bitwise/conservation/dt/blow-up cases plus parity with
the oracle. Compiled here with g++ against libhgks_b200.so."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "native", "test_dropin.cpp")
BIN = os.path.join(ROOT, "tests", "native", "_build", "test_dropin")


def build_dropin_test():
    from paper_2202_13821_b200 import build as B
    B.build()
    import oracle
    oracle.build(ref=False)
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"), SRC,
           "-L", os.path.join(ROOT, "paper_2202_13821_b200"), "-lhgks_b200",
           "-L", os.path.join(ROOT, "oracle", "_build"), "-lhgks_oracle",
           "-Wl,-rpath,$ORIGIN/../../../paper_2202_13821_b200", "-Wl,-rpath,$ORIGIN/../../../oracle/_build",
           "-o", BIN]
    subprocess.run(cmd, check=True)
    return BIN


def test_dropin_header_compiles():
    """CPU: the header and the reference-shaped test program build and link."""
    assert os.path.exists(build_dropin_test())


@pytest.mark.gpu
def test_dropin_suite_on_gpu(hgks):
    binpath = build_dropin_test()
    r = subprocess.run([binpath], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " 0 failed" in r.stdout
