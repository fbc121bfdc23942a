"""e2e host-vector step timing vs z-chunk count: python tools/e2e_probe.py [n] [chunks...]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2202_13821_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
chunks = [int(x) for x in sys.argv[2:]] or [1, 16, 32, 64]
r = P.setup_run(P.CaseConfig.named("tgv", n), P.RunOptions(degree=2))
s = r.solver
q_pin = torch.empty(s.ncoeffs, dtype=torch.float64, pin_memory=True)
q = q_pin.numpy()
q[:], _ = s.get_state()
dof = r.mesh.ncells() * s.N * 5
for nch in chunks:
    for _ in range(2):
        s.two_stage_step_host_streamed(q, s.compute_dt(0.15), nch)
    torch.cuda.synchronize()
    k = 6
    t0 = time.perf_counter()
    for _ in range(k):
        s.two_stage_step_host_streamed(q, s.compute_dt(0.15), nch)
    el = (time.perf_counter() - t0) / k
    print(f"chunks {nch:3d}: {el * 1e3:.2f} ms/step  {dof / el:.3e} DOF-upd/s")
