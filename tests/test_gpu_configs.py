"""Coefficient-level parity at the BASELINE.json configurations and on the
persistent multi-tile path (north_star: 1e-10 norm-relative L-inf on the
modal coefficients after N steps).

The checker is the reference itself (oracle/_ref, headers compiled
unmodified), run on all host cores with the SAME dt sequence as the device
(dt itself is compared at 1e-12 every step, SURVEY §8a gotcha 8).

* C1  adv3d P2 16^3, 100 steps                         (BASELINE configs[0])
* C3  TGV Re=1600 P2 64^3, 10 steps; its Ek / epsZeta series to t = 0.5
      against the reference's own run (tests/golden/tgv64_ref.json)
* C4  TGV Re=1600 P2 128^3, 3 steps                     (the headline config)
* TGV P2 32^3 (20 steps) and P3 32^3 (10 steps): every persistent CTA walks
  several tiles (the double-buffered prefetch, TileWalk::next and the
  loop-carried cp.async groups that run at 128^3)
* the same path forced at small sizes by capping the persistent grids
  (hgks_set_grid_cap): 1..7 CTAs walk every tile of an 8^3 / 12^3 mesh

Per conserved variable the bar is 1e-8 of the variable's own magnitude
(floored at 1e-10 of the state's: rho*W is identically ~0 in 2-D).
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_STATE = 1e-10
TOL_DT = 1e-12
HERE = os.path.dirname(os.path.abspath(__file__))


def rel(a, b):
    d = np.max(np.abs(b))
    return float(np.max(np.abs(a - b)) / (d if d > 0 else 1.0))


def per_var_ok(q_dev, q_ref, N, tol=1e-8):
    gmax = np.max(np.abs(q_ref))
    worst = 0.0
    for v in range(5):
        a, b = q_dev.reshape(-1, N, 5)[:, :, v], q_ref.reshape(-1, N, 5)[:, :, v]
        den = max(np.max(np.abs(b)), 1e-10 * gmax)
        worst = max(worst, np.max(np.abs(a - b)) / den)
    return worst <= tol, worst


def run_pair(P, O, case, n, degree, steps, grid_cap=0, nonuniform=False):
    """Reference and device from the reference's own projected state, K steps
    with the reference's dt; returns (device state, reference state, worst dt
    mismatch)."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    ref = O.RefRun(case, n, degree, nonuniform=nonuniform, workers=os.cpu_count() or 1)
    q0, _ = ref.get_state()
    cfg = P.CaseConfig.named(case, n)
    cfg.nonuniform = nonuniform
    r = P.setup_run(cfg, P.RunOptions(degree=degree))
    s = r.solver
    if grid_cap:
        s.set_grid_cap(grid_cap)
    s.set_state(q0, 0.0)
    cfl = P.default_cfl(degree)
    worst_dt = 0.0
    for _ in range(steps):
        dt = ref.compute_dt(cfl)
        dt_dev = s.compute_dt(cfl)
        worst_dt = max(worst_dt, abs(dt_dev - dt) / dt)
        ref.step(dt)
        s.step(dt)
    q_dev = s.get_state()[0]
    q_ref = ref.get_state()[0]
    return q_dev, q_ref, worst_dt, s.N


@pytest.mark.parametrize("case,n,degree,steps", [
    ("adv3d", 7, 2, 10),     # odd nx: no TMA view (16-byte strides), cp.async staging
    ("tgv", 9, 3, 5),
    ("adv3d", 16, 2, 100),   # C1
    ("tgv", 32, 2, 20),      # multi-tile per CTA
    ("tgv", 32, 3, 10),      # P3: 3 points per face warp
    ("tgv", 64, 2, 10),      # C3
])
def test_config_state_parity(hgks, oracle_mod, case, n, degree, steps):
    q_dev, q_ref, worst_dt, N = run_pair(hgks, oracle_mod, case, n, degree, steps)
    r = rel(q_dev, q_ref)
    ok, pv = per_var_ok(q_dev, q_ref, N)
    print(f"{case} P{degree} {n}^3 {steps} steps: global {r:.3e} per-var {pv:.3e} dt {worst_dt:.3e}")
    assert worst_dt <= TOL_DT
    assert r <= TOL_STATE
    assert ok


@pytest.mark.slow
def test_c4_tgv128_parity(hgks, oracle_mod):
    """BASELINE C4, the headline config: TGV P2 128^3, 3 steps (~16 s of the
    reference on 16 host threads)."""
    q_dev, q_ref, worst_dt, N = run_pair(hgks, oracle_mod, "tgv", 128, 2, 3)
    r = rel(q_dev, q_ref)
    ok, pv = per_var_ok(q_dev, q_ref, N)
    print(f"tgv P2 128^3 3 steps: global {r:.3e} per-var {pv:.3e} dt {worst_dt:.3e}")
    assert worst_dt <= TOL_DT
    assert r <= TOL_STATE
    assert ok



@pytest.mark.parametrize("case,n,degree,steps", [
    ("adv3d", 32, 2, 20),    # C2's mesh family, nonuniform widths at multi-tile size
    ("adv3d", 16, 3, 10),
    ("vortex2d", 80, 2, 20),  # 2-D mode with several tiles per CTA
    ("adv2d", 64, 3, 10),
])
def test_nonuniform_and_2d_parity(hgks, oracle_mod, case, n, degree, steps):
    """Nonuniform meshes (x = xi + 0.05 sin(pi xi), cases.hpp:50-57) and the
    degenerate 2-D mode at sizes where the persistent CTAs walk several
    tiles, against the reference itself (same dt sequence)."""
    q_dev, q_ref, worst_dt, N = run_pair(hgks, oracle_mod, case, n, degree, steps,
                                         nonuniform=case.startswith("adv"))
    r = rel(q_dev, q_ref)
    ok, pv = per_var_ok(q_dev, q_ref, N)
    print(f"{case} P{degree} n={n} {steps} steps: global {r:.3e} per-var {pv:.3e} dt {worst_dt:.3e}")
    assert worst_dt <= TOL_DT
    assert r <= TOL_STATE
    assert ok


@pytest.mark.parametrize("case,n,degree", [("tgv", 4, 2), ("tgv", 4, 3), ("adv3d", 4, 3), ("adv2d", 4, 2),
                                           ("vortex2d", 4, 3), ("tgv", 5, 2)])
def test_smallest_mesh_parity(hgks, oracle_mod, case, n, degree):
    """The smallest meshes build_mesh accepts (4 cells per axis,
    cases.hpp:60): one partial x tile per row, x boxes wider than the mesh
    (TMA zero fill + the periodic wrap patch), every CTA's tile its own
    neighbour's."""
    q_dev, q_ref, worst_dt, N = run_pair(hgks, oracle_mod, case, n, degree, 5)
    assert worst_dt <= TOL_DT
    assert rel(q_dev, q_ref) <= TOL_STATE

@pytest.mark.parametrize("case,n,degree,cap,nonuni", [
    ("tgv", 8, 2, 1, False),
    ("tgv", 8, 2, 7, False),
    ("tgv", 8, 3, 3, False),
    ("adv3d", 12, 2, 5, True),
    ("adv3d", 8, 1, 2, False),
    ("vortex2d", 12, 2, 3, False),
])
def test_persistent_multitile_capped_grid(hgks, oracle_mod, case, n, degree, cap, nonuni):
    """Capped persistent grids: each CTA walks many tiles (tile stride =
    grid), so the prefetch / TileWalk / cp.async group pipeline is exercised
    at sizes the reference finishes instantly."""
    P, O = hgks, oracle_mod
    if degree == 1:  # P1 is unpinned: the C restatement is the checker
        o = O.Oracle(case, n, degree, nonuniform=nonuni)
        cfg = P.CaseConfig.named(case, n)
        cfg.nonuniform = nonuni
        r = P.setup_run(cfg, P.RunOptions(degree=degree))
        r.solver.set_grid_cap(cap)
        r.solver.set_state(o.state.copy(), 0.0)
        for _ in range(5):
            dt = o.compute_dt(0.09)
            o.step(dt)
            r.solver.step(dt)
        assert rel(r.solver.get_state()[0], o.state) <= TOL_STATE
        return
    q_dev, q_ref, worst_dt, N = run_pair(P, O, case, n, degree, 5, grid_cap=cap, nonuniform=nonuni)
    assert worst_dt <= TOL_DT
    assert rel(q_dev, q_ref) <= TOL_STATE
    assert per_var_ok(q_dev, q_ref, N)[0]


def test_capped_grid_bitwise_equal_uncapped(hgks):
    """The tile walk does not change the arithmetic: capped and uncapped grids
    give the same bits (TGV P2 16^3, 3 steps)."""
    P = hgks
    out = []
    for cap in (0, 1, 13):
        r = P.setup_run(P.CaseConfig.named("tgv", 16), P.RunOptions(degree=2))
        r.solver.set_grid_cap(cap)
        for _ in range(3):
            r.solver.step(r.solver.compute_dt(0.15))
        out.append(r.solver.get_state()[0])
    assert np.array_equal(out[0], out[1]) and np.array_equal(out[0], out[2])


def test_c3_tgv64_series_matches_reference(hgks):
    """BASELINE C3: TGV P2 64^3 to t = 0.5 with records every 0.05 through the
    device-resident advance loop, against the reference's own run: the same
    step count, record times, Ek and epsZeta (and epsEk from the series)."""
    P = hgks
    path = os.path.join(HERE, "golden", "tgv64_ref.json")
    g = json.load(open(path))
    r = P.run_case(P.CaseConfig.named("tgv", 64), P.RunOptions(degree=2, t_end=g["t_end"], record_interval=0.05))
    assert r.steps == g["steps"]
    ref = np.array(g["records_t_Ek_epsEk_epsZeta"])
    mine = np.array([[x.t, x.Ek, x.epsEk, x.epsZeta] for x in r.records])
    assert mine.shape == ref.shape
    assert np.max(np.abs(mine[:, 0] - ref[:, 0])) <= 1e-12
    assert np.max(np.abs(mine[:, 1] - ref[:, 1]) / np.abs(ref[:, 1])) <= 1e-10
    assert np.max(np.abs(mine[:, 2] - ref[:, 2]) / np.max(np.abs(ref[:, 2]))) <= 1e-6
    assert np.max(np.abs(mine[:, 3] - ref[:, 3]) / np.abs(ref[:, 3])) <= 1e-9
    q = r.solver.get_state()[0].reshape(-1, r.solver.N, 5)
    l2 = np.array([np.sqrt(np.sum(q[:, n, v] ** 2)) for n in range(r.solver.N) for v in range(5)])
    ref_l2 = np.array(g["final_state"]["per_comp_l2"])
    assert np.max(np.abs(l2 - ref_l2)) <= 1e-10 * np.max(ref_l2)


# ------------------------------------------------ device-resident advance loop
def test_device_loop_equals_host_steps(hgks):
    """hgks_advance_records (dt on the device, CUDA graphs, one-step-ahead
    launches) gives the bits of the host-driven compute_dt + step loop."""
    P = hgks
    a = P.setup_run(P.CaseConfig.named("tgv", 16), P.RunOptions(degree=2))
    b = P.setup_run(P.CaseConfig.named("tgv", 16), P.RunOptions(degree=2))
    for _ in range(7):
        a.solver.step(a.solver.compute_dt(0.15))
    n = b.solver.advance_records(1e9, 0.15, max_steps=7)
    assert n == 7
    assert a.solver.time == b.solver.time
    assert np.array_equal(a.solver.get_state()[0], b.solver.get_state()[0])
    # and without graphs (the same enqueue path, launched eagerly)
    c = P.setup_run(P.CaseConfig.named("tgv", 16), P.RunOptions(degree=2))
    c.solver.set_graphs(False)
    c.solver.advance_records(1e9, 0.15, max_steps=7)
    assert np.array_equal(a.solver.get_state()[0], c.solver.get_state()[0])


def test_device_loop_records_and_clipping(hgks, oracle_mod):
    """advance with records on the device: steps land exactly on the record
    times and t_end, the step count and the records equal the reference's
    advance (TGV P2 8^3 to t = 0.2)."""
    P, O = hgks, oracle_mod
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    ref = O.RefRun("tgv", 8, 2, workers=4)
    steps_ref, rec_ref = ref.advance(0.2, cfl=0.15, record_interval=0.05)
    r = P.run_case(P.CaseConfig.named("tgv", 8), P.RunOptions(degree=2, t_end=0.2, record_interval=0.05))
    assert r.steps == steps_ref
    mine = np.array([[x.t, x.Ek, x.epsEk, x.epsZeta] for x in r.records])
    assert mine.shape == rec_ref.shape
    assert np.max(np.abs(mine[:, 0] - rec_ref[:, 0])) <= 1e-14
    assert np.max(np.abs(mine[:, 1] - rec_ref[:, 1]) / rec_ref[:, 1]) <= 1e-12
    assert rel(r.solver.get_state()[0], ref.get_state()[0]) <= TOL_STATE


def test_device_loop_blowup_leaves_qn(hgks, oracle_mod):
    """A state error inside the device loop: the reference's message (item,
    value) with " at t=<t>", and the solver holds q^n of the failing step."""
    P, O = hgks, oracle_mod
    cfg = P.CaseConfig.named("adv3d", 6)
    r = P.setup_run(cfg, P.RunOptions(degree=2))
    q = r.solver.get_state()[0].reshape(-1, r.solver.N, 5).copy()
    q[2, 0, 0], q[2, 0, 1], q[2, 0, 4] = 1.0, 10.0, 1.0
    q = q.ravel()
    r.solver.set_state(q, 0.0)
    with pytest.raises((P.InvalidStateError, P.NonPositiveDtError)) as e:
        r.solver.advance_records(0.5, 0.15, dt_fixed=1e-3, max_steps=10)
    if isinstance(e.value, P.InvalidStateError):
        assert "pressure" in str(e.value) and " at t=0.000000" in str(e.value)
        o = O.Oracle("adv3d", 6, 2)
        o.set_state(q)
        with pytest.raises(O.OracleError) as eo:
            o.residual(1e-3)
        assert e.value.item == eo.value.item
    assert np.array_equal(r.solver.get_state()[0], q)
    assert r.solver.time == 0.0


def test_streamed_step_failure_restores_q(hgks):
    """hgks_two_stage_step_host_streamed leaves q untouched on a state error
    (integrator.hpp:72-74 semantics)."""
    P = hgks
    r = P.setup_run(P.CaseConfig.named("adv3d", 16), P.RunOptions(degree=2))
    q = r.solver.get_state()[0].reshape(-1, r.solver.N, 5).copy()
    q[700, 0, 0], q[700, 0, 1], q[700, 0, 4] = 1.0, 10.0, 1.0
    q = np.ascontiguousarray(q.ravel())
    before = q.copy()
    with pytest.raises(P.InvalidStateError):
        r.solver.two_stage_step_host_streamed(q, 1e-3, 4)
    assert np.array_equal(q, before)


# ------------------------------------------------ in-library NCCL data plane
def test_nccl_self_ring_bitwise(hgks):
    """hgks_attach_nccl with world = 1: the slab is its own z neighbour, so the
    halo send/recv, the device dt / error-key all-reduces and the overlapped
    boundary faces all run through NCCL on one GPU; the result equals the
    single-slab periodic wrap bit for bit (host-dt steps and the graph loop)."""
    P = hgks
    a = P.setup_run(P.CaseConfig.named("tgv", 16), P.RunOptions(degree=2))
    b = P.setup_run(P.CaseConfig.named("tgv", 16), P.RunOptions(degree=2))
    b.solver.attach_nccl(P.Solver.nccl_unique_id(), 0, 1)
    for _ in range(3):
        dta = a.solver.compute_dt(0.15)
        dtb = b.solver.compute_dt(0.15)
        assert dta == dtb
        a.solver.step(dta)
        b.solver.step(dtb)
    assert np.array_equal(a.solver.get_state()[0], b.solver.get_state()[0])
    a.solver.advance_records(1e9, 0.15, max_steps=4)
    b.solver.advance_records(1e9, 0.15, max_steps=4)
    assert np.array_equal(a.solver.get_state()[0], b.solver.get_state()[0])
    assert np.allclose(b.solver.slab_reduce_sum([1.5, -2.0]), [1.5, -2.0])


# ------------------------------------------------ race shaker (no racecheck here)
@pytest.mark.parametrize("case,n,degree,cap", [("tgv", 8, 2, 2), ("tgv", 8, 3, 2), ("adv3d", 12, 1, 3),
                                               ("vortex2d", 12, 2, 2), ("tgv", 16, 2, 0)])
def test_race_shaker_bitwise(hgks, case, n, degree, cap):
    """compute-sanitizer is closed on this GPU pool, so races are hunted by
    perturbation: pseudo-random per-warp sleeps before every cp.async wait and
    barrier (hgks_set_race_shake) must not change a single bit of the
    residual, the faces, the host-dt steps or the device loop."""
    P = hgks
    cfl = P.default_cfl(degree)
    outs = []
    for seed in (0, 1, 7, 12345):
        r = P.setup_run(P.CaseConfig.named(case, n), P.RunOptions(degree=degree))
        s = r.solver
        s.set_grid_cap(cap)
        s.set_race_shake(seed)
        res = s.residual(s.compute_dt(cfl), faces=True)
        s.step(s.compute_dt(cfl))
        s.advance_records(1e9, cfl, max_steps=2)
        outs.append([res["R"], res["Rt"], *res["faces"], s.get_state()[0]])
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("case,n,degree,cap", [("tgv", 16, 2, 0), ("tgv", 8, 2, 3), ("tgv", 8, 3, 2),
                                               ("adv3d", 12, 1, 2), ("vortex2d", 12, 3, 2), ("adv2d", 10, 2, 0)])
def test_tma_and_cpasync_staging_bitwise(hgks, case, n, degree, cap):
    """The face and cell kernels stage their tiles by TMA (tensor boxes +
    mbarrier) or by per-lane cp.async; the staging moves the same values, so
    residual, faces, host-dt steps and the device loop agree bit for bit
    (including the periodic-x patch of the TMA paths and partial x tiles)."""
    P = hgks
    cfl = P.default_cfl(degree)
    outs = []
    for tma in (True, False):
        r = P.setup_run(P.CaseConfig.named(case, n), P.RunOptions(degree=degree))
        s = r.solver
        s.set_grid_cap(cap)
        s.set_face_tma(tma)
        s.set_cell_tma(tma)
        res = s.residual(s.compute_dt(cfl), faces=True)
        s.step(s.compute_dt(cfl))
        s.advance_records(1e9, cfl, max_steps=2)
        outs.append([res["R"], res["Rt"], *res["faces"], s.get_state()[0]])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
