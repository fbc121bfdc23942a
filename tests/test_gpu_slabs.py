"""z-slab decomposition on ONE GPU: 1, 2 and 4 slabs driven in one process
through the split-phase step (hgks_step_phase) with device-to-device halo
copies between slab solvers. The gate of SURVEY §8e: coefficients bitwise
identical to the single-slab run (the analogue of test_runtime.cpp:80-115).
No kernel waits on another: each phase is launched only after the halos it
needs were copied."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def run_slabs(P, slabs, cfg, degree, world, steps, cfl):
    import torch

    mesh = P.build_mesh(cfg)
    scheme = P.Scheme.make(degree, cfg.dim, P.GasModel.make(cfg.gamma, cfg.viscosity()))
    parts = slabs.slab_partition(mesh.nz, world)
    sol = []
    for zb, zc in parts:
        s = P.Solver(mesh, scheme, 0, zb, zc if world > 1 else 0)
        s.project_case(cfg.name)
        sol.append(s)
    nb = sol[0].halo_bytes()
    views = [[slabs.device_view(p, nb, 0) for p in s.halo_buffers()] for s in sol]
    dts = []
    for _ in range(steps):
        dt = min(s.compute_dt(cfl) for s in sol)
        dts.append(dt)
        for phase in (0, 1):
            if world > 1:
                for s in sol:
                    s.halo_pack(phase)
                    s.synchronize()
                for r in range(world):
                    lo, up = slabs.ring_neighbors(r, world)
                    views[r][2].copy_(views[lo][1])  # recv_lo <- lower's top layer
                    views[r][3].copy_(views[up][0])  # recv_hi <- upper's bottom layer
                torch.cuda.synchronize()
                for s in sol:
                    s.halo_unpack(phase)
            for s in sol:
                s.step_phase(dt, phase)
            for s in sol:
                s.synchronize()
        for s in sol:
            s.step_phase(dt, 2)
    q = np.concatenate([s.get_state()[0] for s in sol])
    return q, dts


@pytest.mark.parametrize("case,n,degree", [("tgv", 8, 2), ("adv3d", 8, 2), ("tgv", 8, 3)])
def test_slabs_bitwise_identical(hgks, case, n, degree):
    P = hgks
    from paper_2202_13821_b200 import slabs
    cfg = P.CaseConfig.named(case, n)
    cfl = P.default_cfl(degree)
    q1, d1 = run_slabs(P, slabs, cfg, degree, 1, 3, cfl)
    # the single-slab split-phase path equals the fused hgks_step path
    r = P.setup_run(cfg, P.RunOptions(degree=degree))
    for d in d1:
        r.solver.step(d)
    assert np.array_equal(r.solver.get_state()[0], q1)
    for world in (2, 4):
        qw, dw = run_slabs(P, slabs, cfg, degree, world, 3, cfl)
        assert dw == d1
        assert np.array_equal(qw, q1), f"world={world}"


def test_slab_flux_count_owned_only(hgks):
    from paper_2202_13821_b200 import slabs
    """Redundant boundary faces are not counted (SURVEY §8a gotcha 9)."""
    P = hgks
    cfg = P.CaseConfig.named("adv3d", 8)
    mesh = P.build_mesh(cfg)
    scheme = P.Scheme.make(2, 3, P.GasModel.make(1.4))
    s = P.Solver(mesh, scheme, 0, 2, 4)
    s.project_case("adv3d")
    s.set_count_fluxes(True)
    # multi-slab residual needs ghosts: a self-wrap exchange keeps them physical
    # (values are irrelevant for the count, but must be valid states)
    views = [slabs.device_view(p, s.halo_bytes(), 0) for p in s.halo_buffers()]

    def self_wrap(solver, which):
        views[2].copy_(views[1])
        views[3].copy_(views[0])

    s.set_halo_exchange(self_wrap)
    s.residual(1e-3)
    assert s.flux_evaluations() == 8 * 8 * 4 * sum(s.face_points(a) for a in range(3))
