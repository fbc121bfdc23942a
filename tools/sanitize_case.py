"""Small multi-tile workload for compute-sanitizer (racecheck / synccheck /
memcheck): every kernel family of the step path on meshes where capped
persistent grids make each CTA walk many tiles.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2202_13821_b200 as P  # noqa: E402


def main():
    for case, n, deg, cap in [("tgv", 8, 2, 2), ("tgv", 6, 3, 2), ("adv3d", 8, 1, 2), ("vortex2d", 8, 2, 2)]:
        r = P.setup_run(P.CaseConfig.named(case, n), P.RunOptions(degree=deg))
        s = r.solver
        s.set_grid_cap(cap)
        cfl = P.default_cfl(deg)
        s.residual(s.compute_dt(cfl), faces=True)          # MODE_RESIDUAL
        s.step(s.compute_dt(cfl))                          # stage 1 / stage 2
        s.advance_records(1e9, cfl, max_steps=2)           # device loop (graphs)
        q = np.ascontiguousarray(s.get_state()[0])
        s.two_stage_step_host_streamed(q, s.compute_dt(cfl), 2)
        print(case, n, deg, "ok", flush=True)


if __name__ == "__main__":
    main()
