"""Compute-side cost of the z-slab decomposition, measured on ONE GPU without
running ranks concurrently: TGV P2 128^3 cut into world = 1, 2, 4, 8 slabs,
each slab stepped in turn through the split-phase step (hgks_step_phase) with
device-to-device halo copies (no kernel waits on another). Per slab: the
CUDA-event time of its face passes and cell kernels per step; per world: the
slowest slab's kernel time is what each GPU would spend per step, so

    compute efficiency = T(1 slab) / (world * T(slowest slab))

measures what the decomposition itself costs (the redundant top z-face
layer, smaller grids, the extra ghost traffic) before any communication.

    python tools/slab_overhead.py [n] [steps]   -> profiles/r02/slab_overhead.json
"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2202_13821_b200 as P  # noqa: E402
from paper_2202_13821_b200 import slabs  # noqa: E402


def run(world, n, steps):
    cfg = P.CaseConfig.named("tgv", n)
    mesh = P.build_mesh(cfg)
    scheme = P.Scheme.make(2, 3, P.GasModel.make(cfg.gamma, cfg.viscosity()))
    sol = []
    for zb, zc in slabs.slab_partition(n, world):
        s = P.Solver(mesh, scheme, 0, zb, zc if world > 1 else 0)
        s.project_case("tgv")
        s.set_kernel_timing(True)
        sol.append(s)
    nb = sol[0].halo_bytes()
    views = [[slabs.device_view(p, nb, 0) for p in s.halo_buffers()] for s in sol]
    per_slab = [[] for _ in sol]
    for it in range(steps + 2):
        dt = min(s.compute_dt(0.15) for s in sol)
        for phase in (0, 1):
            if world > 1:
                for s in sol:
                    s.halo_pack(phase)
                    s.synchronize()
                for r in range(world):
                    lo, up = slabs.ring_neighbors(r, world)
                    views[r][2].copy_(views[lo][1])
                    views[r][3].copy_(views[up][0])
                torch.cuda.synchronize()
                for s in sol:
                    s.halo_unpack(phase)
            for s in sol:
                s.step_phase(dt, phase)
                s.synchronize()
        for k, s in enumerate(sol):
            s.step_phase(dt, 2)
            f, c = s.kernel_times()
            if it >= 2:
                per_slab[k].append(f + c)
    t = [statistics.median(x) for x in per_slab]
    for s in sol:
        s.close()
    return t


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    res = {"workload": f"tgv Re=1600 P2 {n}^3", "method": __doc__.strip().splitlines()[0], "worlds": {}}
    t1 = None
    for world in (1, 2, 4, 8):
        t = run(world, n, steps)
        tmax = max(t)
        if world == 1:
            t1 = tmax
        res["worlds"][str(world)] = {"slab_kernel_ms": t, "slowest_ms": tmax,
                                     "compute_efficiency": t1 / (world * tmax)}
        print(world, [round(x, 3) for x in t], "eff", round(t1 / (world * tmax), 4), flush=True)
    out = os.path.join(ROOT, "profiles", "r02", "slab_overhead.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
