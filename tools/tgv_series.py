"""TGV P2 n^3 record series (Ek, epsZeta every 0.05) + final state -> gpurun_out/."""
import json, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2202_13821_b200 as P
n = int(sys.argv[1]); t_end = float(sys.argv[2])
cfg = P.CaseConfig.named("tgv", n)
opt = P.RunOptions(degree=2, t_end=t_end, record_interval=0.05)
r = P.run_case(cfg, opt)
q, t = r.solver.get_state()
np.save(f"gpurun_out/tgv_{n}_q.npy", q)
json.dump({"steps": r.steps, "rec": [[x.t, x.Ek, x.epsEk, x.epsZeta] for x in r.records], "t": t},
          open(f"gpurun_out/tgv_{n}.json", "w"))
print("steps", r.steps, "t", t)
