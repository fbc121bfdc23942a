"""The C-ABI boundary (CPU): the library loads, exports exactly what
include/hgks_b200.h declares, and fails loudly — never falls back — when no
GPU is present."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hgks_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(hgks_\w+)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if not n.endswith("_fn")))


@pytest.fixture(scope="module")
def lib():
    from paper_2202_13821_b200 import build as B
    B.build()
    from paper_2202_13821_b200 import _lib
    return _lib


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("hgks_create", "hgks_residual", "hgks_step", "hgks_two_stage_step_host", "hgks_compute_dt",
                 "hgks_apply_inverse_mass", "hgks_last_error"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    L = lib.load()
    names = declared_functions()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert sorted(lib.EXPORTS) == names  # the Python binding covers the whole header


def test_exported_symbols_are_plain_c(lib):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for n in declared_functions():
        assert n in exported  # unmangled: extern "C"


def test_library_is_sm100a(lib):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_fails_loudly(lib):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    import paper_2202_13821_b200 as P
    m = P.build_mesh(P.CaseConfig.named("tgv", 4))
    with pytest.raises(P.CudaError):
        P.Solver(m, P.Scheme.make(2, 3, P.GasModel.make(1.4, 1 / 1600)))


def test_config_errors_name_the_problem(lib):
    import paper_2202_13821_b200 as P
    with pytest.raises(P.ConfigError):
        P.Scheme.make(4, 3, P.GasModel.make(1.4))
    with pytest.raises(P.ConfigError):
        P.Mesh.make([0, 1, 0.5], [0, 1], [0, 1])
    with pytest.raises(P.ConfigError):
        P.CaseConfig.named("nope", 8)
    with pytest.raises(P.ConfigError):
        P.build_mesh(P.CaseConfig.named("tgv", 3))


def test_host_mirror_of_cases():
    """case_axis_nodes / build_mesh (cases.hpp:50-73) agree with the oracle's mesh."""
    import numpy as np

    import oracle as O
    import paper_2202_13821_b200 as P
    if not O.ref_available():
        pytest.skip("reference build not available")
    for case, n, nu in [("tgv", 6, False), ("adv3d", 5, True), ("vortex2d", 6, False)]:
        cfg = P.CaseConfig.named(case, n)
        cfg.nonuniform = nu
        m = P.build_mesh(cfg)
        r = O.RefRun(case, n, 2, nonuniform=nu)
        for a, b in zip((m.xs, m.ys, m.zs), r.nodes()):
            assert np.array_equal(a, b)
