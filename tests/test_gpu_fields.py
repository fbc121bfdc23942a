"""Caller-supplied fields: project(field, ...) and error_norms(..., exact, ...)
(dg.hpp:193-220, :228-266) through the Python mirror (Solver.project_field /
error_norms_field -> hgks_project_samples / hgks_error_norms_samples), checked
against the library's built-in case fields (cases.hpp:78-124) on the same
meshes. The projection points come from numpy's Gauss nodes here and from the
reference-identical host tables in the library, so the bar is 1e-13, not
bitwise."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def adv_field(dim, t=0.0, gamma=1.4):
    def f(x, y, z):
        s = x + y + z - 3.0 * t if dim == 3 else x + y - 2.0 * t
        rho = 1.0 + 0.2 * np.sin(np.pi * s)
        W = 1.0 if dim == 3 else 0.0
        E = 1.0 / (gamma - 1.0) + 0.5 * rho * (2.0 + W * W)
        return np.stack([rho, rho, rho, rho * W, E])
    return f


def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


@pytest.mark.parametrize("case,n,degree,nonuniform", [
    ("adv3d", 8, 2, False), ("adv3d", 8, 2, True), ("adv3d", 6, 3, False), ("adv3d", 8, 1, False),
    ("adv2d", 12, 2, True), ("adv2d", 10, 3, False),
])
def test_project_field_matches_case(hgks, case, n, degree, nonuniform):
    P = hgks
    cfg = P.CaseConfig.named(case, n)
    cfg.nonuniform = nonuniform
    r = P.setup_run(cfg, P.RunOptions(degree=degree))
    s = r.solver
    q_case, _ = s.get_state()
    s.project_field(adv_field(cfg.dim))
    q_field, _ = s.get_state()
    assert rel(q_field, q_case) <= 1e-13
    # a few steps, then the caller-field error norms against the built-in ones
    for _ in range(3):
        s.step(s.compute_dt(0.1))
    t = s.time
    e_case = s.error_norm_sums(case, t)
    e_field = s.error_norms_field(adv_field(cfg.dim, t))
    # norms (sqrt of the sums): the cell-average error (~1e-7 here) is a
    # difference of two near-equal means, so its ulp-level sample differences
    # show at ~1e-11 relative; absolute floor 1e-15 of the O(1) density
    np.testing.assert_allclose(np.sqrt(e_field), np.sqrt(e_case), rtol=1e-10, atol=1e-15)
    s.close()


def test_project_field_on_a_slab(hgks):
    """A z-slab solver samples and projects only its owned layers."""
    P = hgks
    cfg = P.CaseConfig.named("adv3d", 8)
    full = P.setup_run(cfg, P.RunOptions(degree=2)).solver
    q_full, _ = full.get_state()
    slab = P.setup_run(cfg, P.RunOptions(degree=2), z_begin=2, z_count=3).solver
    slab.project_field(adv_field(3))
    q_slab, _ = slab.get_state()
    per = 64 * full.N * 5
    assert rel(q_slab, q_full[2 * per:5 * per]) <= 1e-13
    full.close()
    slab.close()


def test_project_field_rejects_bad_shapes(hgks):
    P = hgks
    r = P.setup_run(P.CaseConfig.named("adv3d", 4), P.RunOptions(degree=2))
    with pytest.raises(P.ConfigError):
        r.solver.project_field(lambda x, y, z: np.stack([x, y, z]))
    r.solver.close()
