"""Large-mesh sanity: TGV P2 n^3 (default 256), a few steps; conservation of
the cell-mean totals and finiteness. python tools/big_probe.py [n] [steps]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2202_13821_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
k = int(sys.argv[2]) if len(sys.argv) > 2 else 3
r = P.setup_run(P.CaseConfig.named("tgv", n), P.RunOptions(degree=2))
s = r.solver
q0 = s.get_state()[0].reshape(-1, s.N, 5)
tot0 = q0[:, 0, :].sum(axis=0)
s.set_kernel_timing(True)
for it in range(k):
    dt = s.compute_dt(0.15)
    t0 = time.time()
    s.step(dt)
    s.synchronize()
    f, c = s.kernel_times()
    print(f"step {it}: dt {dt:.6e} wall {1e3 * (time.time() - t0):.1f} ms face {f:.1f} cell {c:.1f}")
q = s.get_state()[0].reshape(-1, s.N, 5)
tot = q[:, 0, :].sum(axis=0)
print("finite", bool(np.isfinite(q).all()), "mean-total drift", np.abs(tot - tot0) / np.maximum(np.abs(tot0), 1.0))
dof = r.mesh.ncells() * s.N * 5
print(f"{dof:.3e} DOF")
