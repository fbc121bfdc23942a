"""Dump residual, faces and a few device-loop steps of small cases with the
library HGKS_LIB points at (variant A/B: python tools/bitwise_ab.py out.npz),
then compare two dumps: python tools/bitwise_ab.py --cmp a.npz b.npz"""
import sys
import numpy as np
sys.path.insert(0, ".")
if sys.argv[1] == "--cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
    for k in bad:
        d = np.max(np.abs(a[k] - b[k])) / max(np.max(np.abs(b[k])), 1e-300)
        print(f"{k}: differs, norm-rel {d:.3e}")
    print("bitwise identical" if not bad else f"{len(bad)} of {len(a.files)} arrays differ")
    sys.exit(0)
import paper_2202_13821_b200 as P
out = {}
for case, n, deg in (("tgv", 12, 2), ("tgv", 8, 3), ("adv3d", 10, 2), ("adv3d", 8, 1), ("vortex2d", 12, 3), ("tgv", 32, 2)):
    r = P.setup_run(P.CaseConfig.named(case, n), P.RunOptions(degree=deg))
    s = r.solver
    cfl = P.default_cfl(deg)
    res = s.residual(s.compute_dt(cfl), faces=True)
    key = f"{case}{n}p{deg}"
    out[key + "_R"], out[key + "_Rt"] = res["R"], res["Rt"]
    for a, f in enumerate(res["faces"]):
        out[f"{key}_f{a}"] = f
    s.advance_records(1e9, cfl, max_steps=5)
    out[key + "_q"] = s.get_state()[0]
    s.close()
np.savez(sys.argv[1], **out)
print("wrote", sys.argv[1])
