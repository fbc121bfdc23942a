"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference headers compiled by oracle/Makefile
(oracle/_ref/libhgks_ref.so, stock flags: FMA contraction as the reference's
own CMake build would have it) on small cases, and writes .npz fixtures:

  residual_<case>.npz  initial state (setup_run projection), CFL dt,
                       ws.R / ws.Rt / ws.face[0..2] of one residual(), and the
                       state after 3 S2O4 steps with its dt sequence
  kinetics.npz         interface_flux_integrals / smooth_flux_integrals /
                       maxwellian_moments on seeded random states

The reference ships no golden vectors; these pin the oracle and the
CUDA path to the reference's actual outputs. Needs /root/reference (this
container only); the fixtures travel, the script does not need to.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402

CASES = [
    ("adv3d", 4, 2, True),
    ("tgv", 4, 2, False),
    ("tgv", 4, 3, False),
    ("adv2d", 6, 3, True),
    ("vortex2d", 6, 2, False),
]


def case_name(case, n, deg, nonuni):
    return f"residual_{case}_n{n}_p{deg}{'_nu' if nonuni else ''}.npz"


def rand_trace(rng, p0, U, gamma=1.4):
    rho = 1.0 + 0.2 * rng.uniform(-1, 1)
    u = U * rng.uniform(-1, 1, 3)
    p = p0 * (1 + 0.1 * rng.uniform(-1, 1))
    E = p / (gamma - 1) + 0.5 * rho * (u @ u)
    q = np.array([rho, rho * u[0], rho * u[1], rho * u[2], E])
    scale = np.array([rho, rho, rho, rho, E])
    dq = (rng.normal(size=(3, 5)) * scale).ravel()
    return np.concatenate([q, dq])


def main():
    O.build(ref=True)
    for case, n, deg, nonuni in CASES:
        r = O.RefRun(case, n, deg, nonuniform=nonuni, workers=2)
        q0, _ = r.get_state()
        cfl = 0.15 if deg == 2 else 0.09
        dt = r.compute_dt(cfl)
        res = r.residual(dt, faces=True, count=True)
        dts = []
        for _ in range(3):
            d = r.compute_dt(cfl)
            dts.append(d)
            r.step(d)
        q3, t3 = r.get_state()
        xs, ys, zs = r.nodes()
        np.savez_compressed(
            os.path.join(HERE, case_name(case, n, deg, nonuni)),
            case=case, n=n, degree=deg, nonuniform=nonuni, xs=xs, ys=ys, zs=zs, q0=q0, dt=dt,
            R=res["R"], Rt=res["Rt"], face0=res["faces"][0], face1=res["faces"][1],
            face2=res["faces"][2], flux_evaluations=res["flux_evaluations"], dts=np.array(dts),
            q3=q3, t3=t3)
    rng = np.random.default_rng(20220228)
    regimes = [(71.4, 1.0, 6.25e-4 / 71.4, 6.7e-4), (1.0, 1.0, 0.0, 0.01), (1.0, 1.0, 0.005, 0.01),
               (1.0, 0.5, 0.01, 0.01), (1.0, 2.0, 1e-3, 0.02)]
    TL, TR, TAU, DT, FF, FH = [], [], [], [], [], []
    ST, SMU, SA, SF, SH = [], [], [], [], []
    PR, MOM = [], []
    for p0, U, tau, dt in regimes:
        for _ in range(24):
            tl, tr = rand_trace(rng, p0, U), rand_trace(rng, p0, U)
            f, h = O.ref_interface_flux(tl, tr, 1.4, tau, dt)
            TL.append(tl); TR.append(tr); TAU.append(tau); DT.append(dt); FF.append(f); FH.append(h)
            t = rand_trace(rng, p0, U)
            mu = tau * p0
            rho = t[0]
            p = 0.4 * (t[4] - 0.5 * (t[1:4] @ t[1:4]) / rho)
            tau_s = mu / p if mu > 0 else 0.0
            for ax in range(3):
                f, h = O.ref_smooth_flux(t, 1.4, tau_s, dt, ax)
                ST.append(t); SMU.append(mu); SA.append(ax); SF.append(f); SH.append(h)
            prim = np.array([t[0], t[1] / t[0], t[2] / t[0], t[3] / t[0], 0.5 * t[0] / p])
            PR.append(prim); MOM.append(O.ref_moments(prim, 1.4))
    np.savez_compressed(os.path.join(HERE, "kinetics.npz"), tl=np.array(TL), tr=np.array(TR), tau=np.array(TAU),
                        dt=np.array(DT), full=np.array(FF), half=np.array(FH), st=np.array(ST), smu=np.array(SMU),
                        sdt=np.repeat(np.array(DT), 3), saxis=np.array(SA), sfull=np.array(SF), shalf=np.array(SH),
                        prim=np.array(PR), moments=np.array(MOM), gamma=1.4)
    print("wrote", sorted(f for f in os.listdir(HERE) if f.endswith(".npz")))


if __name__ == "__main__":
    main()
