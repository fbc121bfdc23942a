"""Build the reference's own doctest suites UNMODIFIED against the drop-in
(TEST INFRASTRUCTURE).

The sources stay where they are (/root/reference/proj/tests/*.cpp, never
copied); they are compiled with
    -I tests/native/doctest_shim      (their <doctest.h>; the vendored one is absent)
    -I include/hgks_b200/compat       ("hgks/*.hpp" -> the B200 drop-in headers)
    -I include
and linked against libhgks_b200.so. The binaries land in
tests/native/_build/ref_<suite> (git-ignored; they travel to the GPU box with
the snapshot, where /root/reference does not exist) and run there under
tests/test_gpu_ref_suites.py.
"""
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF_TESTS = os.environ.get("REF_TESTS", "/root/reference/proj/tests")
OUT = os.path.join(ROOT, "tests", "native", "_build")
# the suites whose subject is the solver interface the drop-in replaces
# (runtime, solver loop, integrator, cases/diagnostics, discretization +
# residual); test_kinetics / test_flux exercise the reference's own host
# kinetics functions, test_config its CLI config loader (out of scope)
SUITES = ["test_runtime", "test_solver", "test_integrator", "test_cases", "test_discretization"]


def binary(suite):
    return os.path.join(OUT, "ref_" + suite)


def sources_present():
    return all(os.path.exists(os.path.join(REF_TESTS, s + ".cpp")) for s in SUITES)


def build(suites=SUITES):
    """Compile each suite (needs the reference tree: this container only)."""
    os.makedirs(OUT, exist_ok=True)
    lib_dir = os.path.join(ROOT, "paper_2202_13821_b200")

    def one(s):
        cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "tests", "native", "doctest_shim"),
               "-I", os.path.join(ROOT, "include", "hgks_b200", "compat"), "-I", os.path.join(ROOT, "include"),
               os.path.join(REF_TESTS, s + ".cpp"), "-L", lib_dir, "-lhgks_b200",
               "-Wl,-rpath,$ORIGIN/../../../paper_2202_13821_b200", "-pthread", "-o", binary(s)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"{s} failed to compile against the drop-in:\n{r.stderr[-3000:]}")
        return binary(s)

    with ThreadPoolExecutor(max_workers=len(suites)) as ex:
        return list(ex.map(one, suites))
