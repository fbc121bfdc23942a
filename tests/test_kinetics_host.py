"""The product's restructured kinetics (csrc/hgks_kinetics.cuh, the exact
__host__ __device__ code the kernels run) compiled for the CPU and checked
against the reference's outputs (golden vectors) and the reference's own
flux property tests (proj/tests/test_flux.cpp). CPU only.
"""
import ctypes
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
_dp = ctypes.POINTER(ctypes.c_double)
GAMMA = 1.4


def P(a):
    return a.ctypes.data_as(_dp)


def lin(full, half, dt):
    """flux_linearize (flux.hpp:180-189)."""
    return (4 * half - full) / dt, (full - 2 * half) * 4 / dt ** 2


def iface(H, tl, tr, tau, dt):
    tl, tr = np.ascontiguousarray(tl, dtype=float), np.ascontiguousarray(tr, dtype=float)
    F, Ft = np.zeros(5), np.zeros(5)
    st, bad = ctypes.c_int(), ctypes.c_double()
    rc = H.hk_interface_flux(P(tl), P(tr), ctypes.c_double(GAMMA), ctypes.c_double(tau), ctypes.c_double(dt),
                             P(F), P(Ft), ctypes.byref(st), ctypes.byref(bad))
    return rc, F, Ft, st.value, bad.value


def smooth(H, t, mu):
    t = np.ascontiguousarray(t, dtype=float)
    out = np.zeros(30)
    bad = ctypes.c_double()
    rc = H.hk_smooth_flux(P(t), ctypes.c_double(GAMMA), ctypes.c_double(mu), P(out), ctypes.byref(bad))
    return rc, out.reshape(3, 10)


def cons(rho, U, V, W, lam):
    p = 0.5 * rho / lam
    return np.array([rho, rho * U, rho * V, rho * W, p / (GAMMA - 1) + 0.5 * rho * (U * U + V * V + W * W)])


def rel(a, b):
    d = np.max(np.abs(b))
    return float(np.max(np.abs(a - b)) / (d if d > 0 else 1.0))


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(HERE, "golden", "kinetics.npz"))


def test_interface_flux_vs_reference_golden(kin_host, golden):
    g = golden
    for i in range(len(g["tau"])):
        rc, F, Ft, _, _ = iface(kin_host, g["tl"][i], g["tr"][i], g["tau"][i], g["dt"][i])
        assert rc == 0
        Fr, Ftr = lin(g["full"][i], g["half"][i], g["dt"][i])
        assert rel(F, Fr) <= 1e-13
        # Ft: the reference's If - 2 Ih loses ~4 eps/dt relative to |F|
        assert np.max(np.abs(Ft - Ftr)) <= 1e-10 * max(np.max(np.abs(Ftr)), np.max(np.abs(Fr)))


def test_smooth_flux_vs_reference_golden(kin_host, golden):
    g = golden
    for i in range(len(g["saxis"])):
        rc, out = smooth(kin_host, g["st"][i], g["smu"][i])
        assert rc == 0
        ax = int(g["saxis"][i])
        Fr, Ftr = lin(g["sfull"][i], g["shalf"][i], g["sdt"][i])
        assert rel(out[ax, :5], Fr) <= 1e-13
        assert np.max(np.abs(out[ax, 5:] - Ftr)) <= 1e-10 * max(np.max(np.abs(Ftr)), np.max(np.abs(Fr)))


def test_free_stream_exactness(kin_host):
    """test_flux.cpp:185-196: identical uniform traces give the Euler flux."""
    w = (1.4, 0.6, -0.3, 0.8, 0.7)
    q = cons(*w)
    t = np.concatenate([q, np.zeros(15)])
    p = 0.5 * w[0] / w[4]
    euler = np.array([q[0] * w[1], q[1] * w[1] + p, q[2] * w[1], q[3] * w[1], (q[4] + p) * w[1]])
    for tau in (0.0, 0.01, 10.0):
        rc, F, Ft, _, _ = iface(kin_host, t, t, tau, 0.12)
        assert rc == 0
        assert np.max(np.abs(F - euler)) <= 1e-12 * np.max(np.abs(euler))
        assert np.max(np.abs(Ft)) <= 1e-11 * np.max(np.abs(euler))


def test_tau0_equals_smooth(kin_host):
    """test_flux.cpp:198-212 and :271-283: identical smooth traces -> the
    interface flux equals the smooth in-cell flux (tau = 0 and tau > 0)."""
    q = cons(1.1, 0.5, 0.2, -0.1, 0.9)
    dq = np.array([[0.15, 0.08, -0.02, 0.05, 0.2], [-0.06, 0.01, 0.09, 0.0, 0.04],
                   [0.02, -0.03, 0.01, 0.07, -0.05]]).ravel()
    t = np.concatenate([q, dq])
    rc, F, Ft, _, _ = iface(kin_host, t, t, 0.0, 0.08)
    rc2, out = smooth(kin_host, t, 0.0)
    assert rc == 0 and rc2 == 0
    assert np.max(np.abs(F - out[0, :5])) <= 1e-12 * np.max(np.abs(F))
    assert np.max(np.abs(Ft - out[0, 5:])) <= 1e-11 * np.max(np.abs(F))
    # tau > 0, identical traces: the Heaviside halves recombine (test_flux.cpp:271-283)
    tau = 0.02
    p = 0.5 * 1.1 / 0.9
    rc, F, Ft, _, _ = iface(kin_host, t, t, tau, 0.05)
    rc2, out = smooth(kin_host, t, tau * p)
    assert np.max(np.abs(F - out[0, :5])) <= 1e-12 * np.max(np.abs(F))


def test_galilean_reflection(kin_host):
    """test_flux.cpp:228-269: mirroring u -> -u and swapping sides negates the mass flux."""
    rng = np.random.default_rng(41)
    for _ in range(20):
        wl, wr = (1.2, 0.4, 0.1, -0.2, 0.8), (0.9, 0.2, -0.3, 0.1, 1.1)
        dl, dr = rng.uniform(-0.3, 0.3, (3, 5)), rng.uniform(-0.3, 0.3, (3, 5))

        def mirror(w, d):
            m = cons(w[0], -w[1], w[2], w[3], w[4])
            d = d.copy()
            d[:, 1] *= -1
            d[0] *= -1
            return np.concatenate([m, d.ravel()])

        L = np.concatenate([cons(*wl), dl.ravel()])
        R = np.concatenate([cons(*wr), dr.ravel()])
        _, F, Ft, _, _ = iface(kin_host, L, R, 0.02, 0.05)
        _, M, Mt, _, _ = iface(kin_host, mirror(wr, dr), mirror(wl, dl), 0.02, 0.05)
        assert M[0] == pytest.approx(-F[0], rel=1e-11, abs=1e-13)
        assert Mt[0] == pytest.approx(-Ft[0], rel=1e-9, abs=1e-11)


def test_first_order_in_tau(kin_host):
    """test_flux.cpp:285-306: interface flux -> inviscid smooth flux at O(tau)."""
    q = cons(1.05, 0.4, 0.15, -0.2, 0.85)
    dq = np.array([[0.1, 0.05, -0.01, 0.04, 0.12], [-0.03, 0.02, 0.06, 0.01, 0.02],
                   [0.01, -0.02, 0.03, 0.05, -0.04]]).ravel()
    t = np.concatenate([q, dq])
    _, s0 = smooth(kin_host, t, 0.0)
    # integral form over [0, dt]: F dt + Ft dt^2/2
    dt = 0.05
    S0 = s0[0, :5] * dt + s0[0, 5:] * dt * dt / 2

    def diff(tau):
        _, F, Ft, _, _ = iface(kin_host, t, t, tau, dt)
        return np.max(np.abs(F * dt + Ft * dt * dt / 2 - S0))

    d1, d2, d4 = diff(1e-3), diff(5e-4), diff(2.5e-4)
    assert d2 / d1 == pytest.approx(0.5, rel=0.2)
    assert d4 / d2 == pytest.approx(0.5, rel=0.2)


def test_time_weights_limits(kin_host):
    """flux.hpp:32-48 via closed-form weights: tau=0 limits, continuity, clamp."""
    w = np.zeros(12)
    kin_host.hk_time_weights(ctypes.c_double(0.0), ctypes.c_double(0.2), P(w))
    assert list(w) == [1.0, 0.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0]
    w2 = np.zeros(12)
    kin_host.hk_time_weights(ctypes.c_double(1e-9), ctypes.c_double(0.2), P(w2))
    assert np.max(np.abs(w2 - w)) <= 1e-7
    w3 = np.zeros(12)
    kin_host.hk_time_weights(ctypes.c_double(1e-6), ctypes.c_double(1.0), P(w3))  # dt/tau >> 700
    assert np.all(np.isfinite(w3))


def test_state_errors_and_order(kin_host):
    """core.hpp:76-82 check order: left density, left pressure, right, merged."""
    good = np.concatenate([cons(1.0, 0.1, 0, 0, 0.5), np.zeros(15)])
    bad_rho = good.copy()
    bad_rho[0] = -1.0
    bad_p = good.copy()
    bad_p[4] = 0.0
    rc, *_, st, val = iface(kin_host, bad_rho, good, 0.0, 0.1)
    assert (rc, st, val) == (1, 0, -1.0)
    rc, *_, st, val = iface(kin_host, good, bad_p, 0.0, 0.1)
    assert (rc, st) == (2, 1) and val < 0
    rc, *_, st, _ = iface(kin_host, bad_p, bad_rho, 0.0, 0.1)
    assert (rc, st) == (2, 0)
