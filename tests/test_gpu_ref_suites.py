"""The reference's OWN doctest suites, compiled unmodified against the C++
drop-in (include/hgks_b200/compat/hgks/*.hpp -> hgks_b200/hgks.hpp) and run
on the GPU: the test that a reference C++ caller can switch its include path
and keep calling the solver interface.

Suites: test_runtime, test_solver, test_integrator, test_cases,
test_discretization (/root/reference/proj/tests). Built by
tests/native/ref_suites.py in the container (the reference tree is not on
the GPU box; the binaries travel with the snapshot)."""
import importlib.util
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_spec = importlib.util.spec_from_file_location("_ref_suites", os.path.join(ROOT, "tests", "native", "ref_suites.py"))
RS = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(RS)


@pytest.mark.skipif(not RS.sources_present(), reason="reference test sources not in this container")
def test_reference_suites_compile_against_dropin():
    """CPU: every suite compiles and links against the drop-in headers."""
    from paper_2202_13821_b200 import build as B
    B.build()
    for b in RS.build():
        assert os.path.exists(b)


@pytest.mark.gpu
@pytest.mark.parametrize("suite", RS.SUITES)
def test_reference_suite_passes_on_gpu(hgks, suite):
    binpath = RS.binary(suite)
    if RS.sources_present():
        RS.build([suite])
    assert os.path.exists(binpath), f"{binpath} missing: build() compiles it where /root/reference exists"
    r = subprocess.run([binpath], capture_output=True, text=True, timeout=1200)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
