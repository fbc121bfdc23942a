"""Quick device timing probe: TGV P2 n^3, a few steps, CUDA-event kernel split."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2202_13821_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
deg = int(sys.argv[2]) if len(sys.argv) > 2 else 2
case = sys.argv[3] if len(sys.argv) > 3 else "tgv"
t0 = time.time()
r = P.setup_run(P.CaseConfig.named(case, n), P.RunOptions(degree=deg))
print("setup", time.time() - t0)
s = r.solver
import os
s.set_face_tma(os.environ.get("HGKS_FACE_TMA", "1") != "0")
s.set_cell_tma(os.environ.get("HGKS_CELL_TMA", "1") != "0")
s.set_kernel_timing(True)
dt = s.compute_dt(0.15)
print("dt", dt)
for it in range(6):
    t0 = time.time()
    s.step(dt)
    s.synchronize()
    w = time.time() - t0
    f, c = s.kernel_times()
    dof = r.mesh.ncells() * s.N * 5
    print(f"step {it}: wall {w*1e3:.2f} ms  face {f:.2f} ms  cell {c:.2f} ms  -> {dof/w:.3e} DOF-upd/s (wall)")
