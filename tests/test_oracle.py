"""The oracle itself, pinned before it is trusted (CPU only).

1. The plain-C restatement vs the golden vectors generated from the reference
   build (tests/golden/make_golden.py): projection, compute_dt, residual
   (R, Rt, faces), flux count, 3 S2O4 steps.
2. Bitwise identity of the restatement with the reference compiled with the
   same contraction setting (oracle/_ref/libhgks_ref_nofma.so), when present.
3. The reference's own known answers (test_integrator.cpp, test_cases.cpp,
   test_solver.cpp) replayed on the restatement.
"""
import glob
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "residual_*.npz")))


def rel(a, b):
    d = np.max(np.abs(b))
    return float(np.max(np.abs(a - b)) / (d if d > 0 else 1.0))


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_restatement_matches_golden(oracle_mod, path):
    O = oracle_mod
    g = np.load(path)
    o = O.Oracle(str(g["case"]), int(g["n"]), int(g["degree"]), nonuniform=bool(g["nonuniform"]))
    assert rel(o.state, g["q0"]) <= 1e-14
    deg = int(g["degree"])
    dt = o.compute_dt(0.15 if deg == 2 else 0.09)
    assert abs(dt - float(g["dt"])) <= 1e-14 * dt
    res = o.residual(float(g["dt"]), coeffs=g["q0"], faces=True, count=True)
    assert res["flux_evaluations"] == int(g["flux_evaluations"])
    assert rel(res["R"], g["R"]) <= 1e-12
    assert rel(res["Rt"], g["Rt"]) <= 1e-11  # reference's own If - 2 Ih cancellation
    for a in range(3):
        assert rel(res["faces"][a], g[f"face{a}"]) <= 1e-11
    o.set_state(g["q0"])
    for d in g["dts"]:
        o.step(float(d))
    assert rel(o.state, g["q3"]) <= 1e-13


@pytest.mark.parametrize("case,n,deg,nonuni", [("adv3d", 4, 2, True), ("tgv", 4, 2, False),
                                               ("tgv", 4, 3, False), ("vortex2d", 6, 3, False),
                                               ("adv2d", 6, 2, True)])
def test_restatement_bitwise_vs_reference(oracle_mod, case, n, deg, nonuni):
    O = oracle_mod
    if not os.path.exists(O.REF_NOFMA_SO):
        pytest.skip("reference build (contraction off) not available")
    r = O.RefRun(case, n, deg, nonuniform=nonuni, workers=3, lib="nofma")
    o = O.Oracle(case, n, deg, nonuniform=nonuni)
    q0, _ = r.get_state()
    assert np.array_equal(o.state, q0)
    cfl = 0.15 if deg == 2 else 0.09
    for _ in range(3):
        dt = r.compute_dt(cfl)
        assert dt == o.compute_dt(cfl)
        a, b = r.residual(dt, faces=True), o.residual(dt, faces=True)
        assert np.array_equal(a["R"], b["R"]) and np.array_equal(a["Rt"], b["Rt"])
        for x, y in zip(a["faces"], b["faces"]):
            assert np.array_equal(x, y)
        r.step(dt)
        o.step(dt)
    assert np.array_equal(r.get_state()[0], o.state)


def test_compute_dt_rest_gas_known_answer(oracle_mod):
    """test_integrator.cpp:13-24: dt = 0.15 * 0.1 / sqrt(1.4) for rest gas p = 1."""
    O = oracle_mod
    nodes = np.array([0.0, 0.1, 0.2])
    o = O.Oracle(mesh=(nodes, nodes, nodes), degree=2, dim=3, gamma=1.4, mu=0.0)
    q = np.zeros(o.ncoeffs).reshape(-1, o.N, 5)
    q[:, 0, 0] = 1.0
    q[:, 0, 4] = 1.0 / 0.4
    o.set_state(q.ravel())
    assert o.compute_dt(0.15) == pytest.approx(0.15 * 0.1 / np.sqrt(1.4), rel=1e-12)


def test_tgv_initial_diagnostics(oracle_mod):
    """test_cases.cpp:140-150: Ek(0) = 0.125, epsZeta(0) = 0.75/1600 (to projection accuracy)."""
    O = oracle_mod
    o = O.Oracle("tgv", 8, 2)
    ek, ez = o.tgv_diagnostics()
    assert ek == pytest.approx(0.125, rel=2e-3)
    assert ez == pytest.approx(0.75 / 1600, rel=5e-2)


def test_tgv_first_dt_128(oracle_mod):
    """TGV P2 128^3 first CFL dt = 6.6941e-4 (measured on the reference)."""
    O = oracle_mod
    if not O.ref_available():
        pytest.skip("reference build not available")
    r = O.RefRun("tgv", 32, 2, workers=4)
    # dt scales with h at fixed Mach: 32^3 -> 4x the 128^3 value (to projection accuracy)
    assert r.compute_dt(0.15) / 4 == pytest.approx(6.6941e-4, rel=2e-3)


def test_blowup_error_message_shape(oracle_mod):
    """test_solver.cpp:122-140 / runtime.hpp:37-41: item index + reference message."""
    O = oracle_mod
    o = O.Oracle("adv3d", 6, 2)
    q = o.state.reshape(-1, o.N, 5)
    q[2, 0, 0], q[2, 0, 1], q[2, 0, 4] = 1.0, 10.0, 1.0
    with pytest.raises(O.OracleError) as e:
        o.residual(1e-3)
    assert str(e.value).startswith("item ")
    assert "non-positive pressure: p=" in str(e.value)
    if O.ref_available():
        r = O.RefRun("adv3d", 6, 2, workers=4)
        r.set_state(o.state.copy())
        with pytest.raises(O.RefError) as er:
            r.residual(1e-3)
        assert str(er.value) == str(e.value)


def test_conservation_over_steps(oracle_mod):
    """test_solver.cpp:22-53: totals constant to 1e-12 per step."""
    O = oracle_mod
    o = O.Oracle("adv2d", 8, 2)
    vol = (2.0 / 8) ** 2 * 2.0

    def totals():
        return vol * o.state.reshape(-1, o.N, 5)[:, 0, :].sum(axis=0)

    before = totals()
    for s in range(10):
        o.step(o.compute_dt(0.15))
        assert np.all(np.abs(totals() - before) <= 1e-12 * np.maximum(1.0, np.abs(before)) * (s + 1))
