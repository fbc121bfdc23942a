"""The reference's acceptance criteria (proj/tests/acceptance.cpp:83-252),
replayed on the B200 path: the paper's published convergence tables
 and the Taylor-Green analytics. These runs take hours on
the CPU reference; they take seconds here. Tolerances are the reference's.
"""
import math

import pytest

pytestmark = pytest.mark.gpu


def study(P, case, meshes, **kw):
    return P.solver.convergence_study(case, meshes, P.solver.StudyOptions(**kw))


def test_criterion1_adv2d_p2_paper_table(hgks):
    """acceptance.cpp:83-98: adv2d P2, dt ~ h^2 (safety 0.7): eL1 within 30% of
    the paper and orders within 0.2."""
    P = hgks
    rows = study(P, "adv2d", [8, 16, 32, 64], degree=2, dt_power=2.0, dt_safety=0.7)
    paper_l1 = [1.2632e-2, 1.2982e-3, 1.5215e-4, 1.8633e-5]
    paper_o = [3.28, 3.09, 3.03]
    for r, pl in zip(rows, paper_l1):
        assert 0.7 < r.err.l1 / pl < 1.3, (r.n, r.err.l1, pl)
    for i in range(3):
        o = P.solver.order(rows[i], rows[i + 1], "l1")
        assert abs(o - paper_o[i]) <= 0.2, (i, o)
    # criterion 3 (acceptance.cpp:139-147): cell-average super-convergence
    for i in range(3):
        assert P.solver.order(rows[i], rows[i + 1], "cell_avg") >= 3.9


@pytest.mark.parametrize("degree,nonuniform,l1_16,l1_32,l2_16,l2_32", [
    (2, False, 2.9226e-3, 2.9518e-4, 1.1441e-3, 1.1712e-4),
    (2, True, 3.1274e-3, 3.1367e-4, 1.2335e-3, 1.2516e-4),
    (3, False, 9.0567e-5, 5.6787e-6, 5.3092e-5, 3.3471e-6),
    (3, True, 1.0973e-4, 6.7226e-6, 5.4167e-5, 3.3516e-6),
])
def test_criterion4_adv3d_paper_table(hgks, degree, nonuniform, l1_16, l1_32, l2_16, l2_32):
    """acceptance.cpp:149-182 (BASELINE config C2): 3-D advection, nominal CFL
    steps on 8/16/32^3; L1/L2 orders k+1 +- 0.3 (the paper's orders).

    Magnitudes are pinned to the REFERENCE's own study outputs
    (tests/golden/acceptance_ref.json, make_acceptance_golden.py) at 1e-6:
    the reference itself lands outside acceptance.cpp's 30% band around the
    paper's table for P2 uniform 16^3 (L1 3.896e-3 vs 2.9226e-3, ratio 1.333),
    so the paper ratio is reported, not asserted."""
    import json
    import os
    P = hgks
    rows = study(P, "adv3d", [8, 16, 32], degree=degree, nominal=True, nonuniform=nonuniform)
    target = degree + 1.0
    o1 = P.solver.order(rows[1], rows[2], "l1")
    o2 = P.solver.order(rows[1], rows[2], "l2")
    print(f"P{degree} nonuniform={nonuniform}: orders L1 {o1:.3f} L2 {o2:.3f}; paper ratios "
          f"{rows[1].err.l1 / l1_16:.3f} {rows[2].err.l1 / l1_32:.3f} {rows[1].err.l2 / l2_16:.3f} "
          f"{rows[2].err.l2 / l2_32:.3f}")
    assert abs(o1 - target) <= 0.3
    assert abs(o2 - target) <= 0.3
    gold = os.path.join(os.path.dirname(__file__), "golden", "acceptance_ref.json")
    key = f"adv3d_p{degree}_{'nonuniform' if nonuniform else 'uniform'}"
    ref = json.load(open(gold)).get(key, []) if os.path.exists(gold) else []
    assert ref, f"no reference golden rows for {key}"
    for g in ref:
        mine = next(r for r in rows if r.n == g["n"])
        assert mine.steps == g["steps"]
        for norm in ("l1", "l2", "cell_avg"):
            assert abs(getattr(mine.err, norm) - g[norm]) <= 1e-6 * g[norm], (g["n"], norm)


def test_criterion5_vortex_p2_orders(hgks):
    """acceptance.cpp:184-195: isotropic vortex P2, nominal steps, 20..160^2."""
    P = hgks
    rows = study(P, "vortex2d", [20, 40, 80, 160], degree=2, nominal=True)
    paper = [2.94, 2.82, 2.95]
    for i in range(3):
        o = P.solver.order(rows[i], rows[i + 1], "l1")
        assert abs(o - paper[i]) <= 0.3, (i, o)


def test_criterion6_tgv32_analytics(hgks):
    """acceptance.cpp:206-252: TGV P2 32^3 to t = 10, records every 0.05:
    Ek(0) = 0.125, epsZeta(0) = 4.6875e-4 (2%), and the integrated
    central-difference dissipation matches the Ek drop to 1%.

    The criterion's "Ek monotone" clause is NOT asserted: the reference
    scheme itself (no limiter, under-resolved meshes) gains kinetic energy
    from t ~ 3.5 at 16^3 and 32^3 — test_tgv16_series_matches_reference shows
    the device series is the reference's to 1e-9."""
    P = hgks
    cfg = P.CaseConfig.named("tgv", 32)
    r = P.run_case(cfg, P.RunOptions(degree=2, record_interval=0.05))
    recs = r.records
    assert len(recs) == 201
    assert abs(recs[0].Ek - 0.125) <= 1e-6
    assert abs(recs[0].epsZeta - 4.6875e-4) <= 0.02 * 4.6875e-4
    integral = sum(0.5 * (b.epsEk + a.epsEk) * (b.t - a.t) for a, b in zip(recs, recs[1:]))
    drop = recs[0].Ek - recs[-1].Ek
    assert abs(integral - drop) <= 0.01 * abs(drop)
    assert abs(recs[-1].t - 10.0) <= 1e-9
    assert all(math.isfinite(x.Ek) and math.isfinite(x.epsZeta) for x in recs)


def test_tgv16_series_matches_reference(hgks):
    """1000 S2O4 steps of TGV P2 16^3 (t = 0..5, records every 0.05) against the
    reference's own run (tests/golden/tgv16_ref.json): same step count, Ek and
    epsZeta series, and final-state digest."""
    import json
    import os

    import numpy as np
    P = hgks
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tgv16_ref.json")))
    r = P.run_case(P.CaseConfig.named("tgv", 16), P.RunOptions(degree=2, t_end=5.0, record_interval=0.05))
    assert r.steps == g["steps"]
    ref = np.array(g["records_t_Ek_epsEk_epsZeta"])
    mine = np.array([[x.t, x.Ek, x.epsEk, x.epsZeta] for x in r.records])
    assert mine.shape == ref.shape
    assert np.max(np.abs(mine[:, 0] - ref[:, 0])) <= 1e-12
    assert np.max(np.abs(mine[:, 1] - ref[:, 1]) / np.abs(ref[:, 1])) <= 1e-9
    assert np.max(np.abs(mine[:, 3] - ref[:, 3]) / np.abs(ref[:, 3])) <= 1e-8
    q = r.solver.get_state()[0].reshape(-1, r.solver.N, 5)
    l2 = np.array([np.sqrt(np.sum(q[:, n, v] ** 2)) for n in range(r.solver.N) for v in range(5)])
    ref_l2 = np.array(g["final_state"]["per_comp_l2"])
    assert np.max(np.abs(l2 - ref_l2)) <= 1e-10 * np.max(ref_l2)


def test_error_norms_match_oracle(hgks, oracle_mod):
    """device error_norms (dg.hpp:228-266) vs the oracle after a few steps."""
    P, O = hgks, oracle_mod
    for case, n, deg in [("adv3d", 6, 2), ("vortex2d", 8, 3)]:
        cfg = P.CaseConfig.named(case, n)
        r = P.setup_run(cfg, P.RunOptions(degree=deg))
        o = O.Oracle(case, n, deg)
        r.solver.set_state(o.state.copy(), 0.0)
        for _ in range(3):
            dt = o.compute_dt(0.15 if deg == 2 else 0.09)
            o.step(dt)
            r.solver.step(dt)
        t = r.solver.time
        a = r.solver.error_norms(case, t)
        b = o.error_norms(t)
        for x, y in zip(a, b):
            assert abs(x - y) <= 1e-9 * abs(y)


@pytest.mark.parametrize("degree", [1, 2])
def test_config2_adv3d_sweep_32_64_128(hgks, degree):
    """BASELINE config C2 at its own sizes: the 3-D advection convergence
    sweep at 32^3 / 64^3 / 128^3 with the nominal CFL step (solver.hpp:161-202),
    L1/L2 orders k+1 +- 0.3 on both refinements. The 32^3 P2 row is pinned to
    the reference's own study output (tests/golden/acceptance_ref.json) at 1e-6;
    P1 is the extension degree (no reference run exists to pin it to)."""
    import json
    import os
    P = hgks
    rows = study(P, "adv3d", [32, 64, 128], degree=degree, nominal=True)
    target = degree + 1.0
    for i in range(2):
        for norm in ("l1", "l2"):
            o = P.solver.order(rows[i], rows[i + 1], norm)
            print(f"P{degree} {rows[i].n}->{rows[i + 1].n} {norm} order {o:.3f}")
            if degree == 2:
                assert abs(o - target) <= 0.3, (degree, rows[i].n, norm, o)
            else:  # P1 runs super-convergent on this smooth field (L1 32->64: 2.37)
                assert o >= target - 0.3, (degree, rows[i].n, norm, o)
    if degree == 2:
        gold = os.path.join(os.path.dirname(__file__), "golden", "acceptance_ref.json")
        g = next(r for r in json.load(open(gold))["adv3d_p2_uniform"] if r["n"] == 32)
        assert rows[0].steps == g["steps"]
        for norm in ("l1", "l2", "cell_avg"):
            assert abs(getattr(rows[0].err, norm) - g[norm]) <= 1e-6 * g[norm], norm
