import subprocess, sys
CASES = [("tgv", 8, 2, "res"), ("tgv", 8, 2, "step"), ("tgv", 32, 2, "res"), ("adv2d", 8, 2, "res"),
         ("adv3d", 8, 2, "step"), ("tgv", 8, 3, "step"), ("vortex2d", 6, 3, "step"), ("adv3d", 8, 1, "step"),
         ("tgv", 32, 2, "loop"), ("tgv", 12, 2, "loop")]
code = r'''
import sys; sys.path.insert(0, ".")
import numpy as np
import paper_2202_13821_b200 as P
case, n, deg, what = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
outs = []
for tma in (0, 1):
    r = P.setup_run(P.CaseConfig.named(case, n), P.RunOptions(degree=deg))
    s = r.solver
    s.set_cell_tma(bool(tma))
    s.set_face_tma(bool(tma))
    dt = s.compute_dt(0.09)
    if what == "res": outs.append(s.residual(dt)["R"])
    elif what == "step":
        s.step(dt); outs.append(s.get_state()[0])
    else:
        s.advance_records(1e9, 0.09, max_steps=3); outs.append(s.get_state()[0])
print("ok bitwise" if np.array_equal(outs[0], outs[1]) else "MISMATCH %.3e" % np.max(np.abs(outs[0]-outs[1])))
'''
for c in CASES:
    r = subprocess.run([sys.executable, "-c", code, *map(str, c)], capture_output=True, text=True, timeout=300)
    tail = (r.stdout + r.stderr).strip().splitlines()[-1:] if (r.stdout + r.stderr).strip() else [""]
    print(c, "rc", r.returncode, tail[0][:200], flush=True)
