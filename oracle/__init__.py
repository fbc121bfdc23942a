"""TEST INFRASTRUCTURE ONLY — ctypes access to the two CPU checkers.

* ``Oracle``    — the plain-C restatement (oracle/hgks_oracle.c, built into
  oracle/_build/libhgks_oracle.so).
* ``RefRun``    — the unmodified reference headers compiled in place
  (oracle/ref_driver.cpp -> oracle/_ref/libhgks_ref.so).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this package. The product path (paper_2202_13821_b200) never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libhgks_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhgks_ref.so")
# the reference built with its own CMake flags (-O3 -march=native), for the
# CPU baseline; REF_SO (-march=x86-64-v3) is the portable checker
REF_NATIVE_SO = os.path.join(HERE, "_ref", "libhgks_ref_native.so")
# FMA contraction off: the C restatement's bitwise pin (tests/test_oracle.py)
REF_NOFMA_SO = os.path.join(HERE, "_ref", "libhgks_ref_nofma.so")

_dp = ctypes.POINTER(ctypes.c_double)


def _ptr(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


def build(ref: bool = True) -> None:
    """Compile the oracle (and, when the reference tree is present, oracle/_ref)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if ref and os.path.isdir(os.environ.get("REF_INC", "/root/reference/proj/include")):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


class OracleError(RuntimeError):
    def __init__(self, code, item, value, msg):
        super().__init__(msg)
        self.code, self.item, self.value = code, item, value


class _OrcError(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int), ("item", ctypes.c_int), ("value", ctypes.c_double),
                ("msg", ctypes.c_char * 256)]


_orc = None


def _orc_lib():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        L = ctypes.CDLL(ORACLE_SO)
        L.orc_setup.restype = ctypes.c_void_p
        L.orc_setup.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                ctypes.POINTER(_OrcError)]
        L.orc_create.restype = ctypes.c_void_p
        L.orc_create.argtypes = [ctypes.c_int] * 3 + [_dp] * 3 + [ctypes.c_int, ctypes.c_int,
                                 ctypes.c_double, ctypes.c_double, ctypes.POINTER(_OrcError)]
        L.orc_free.argtypes = [ctypes.c_void_p]
        for f in ("orc_N", "orc_ncells"):
            getattr(L, f).argtypes = [ctypes.c_void_p]
        L.orc_ncoeffs.restype = ctypes.c_long
        L.orc_ncoeffs.argtypes = [ctypes.c_void_p]
        L.orc_state.restype = _dp
        L.orc_state.argtypes = [ctypes.c_void_p]
        L.orc_face_npts.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.orc_residual.argtypes = [ctypes.c_void_p, _dp, ctypes.c_double, _dp, _dp, _dp, _dp, _dp,
                                   ctypes.POINTER(ctypes.c_long), ctypes.POINTER(_OrcError)]
        L.orc_apply_inverse_mass.argtypes = [ctypes.c_void_p, _dp, _dp]
        L.orc_compute_dt.argtypes = [ctypes.c_void_p, ctypes.c_double, _dp, ctypes.POINTER(_OrcError)]
        L.orc_step.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.POINTER(_OrcError)]
        L.orc_tgv_diagnostics.argtypes = [ctypes.c_void_p, _dp]
        L.orc_error_norms.argtypes = [ctypes.c_void_p, ctypes.c_double, _dp]
        L.orc_interface_flux.argtypes = [_dp, _dp, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                         _dp, _dp, ctypes.POINTER(_OrcError)]
        L.orc_smooth_flux.argtypes = [_dp, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_int, _dp, _dp, ctypes.POINTER(_OrcError)]
        L.orc_maxwellian_moments.argtypes = [_dp, ctypes.c_double, _dp]
        _orc = L
    return _orc


def _raise(e: _OrcError):
    raise OracleError(e.code, e.item, e.value, e.msg.decode())


class Oracle:
    """The C restatement: one solver instance (mesh + scheme + AoS state)."""

    def __init__(self, case=None, n=None, degree=2, nonuniform=False, *, mesh=None, dim=3,
                 gamma=1.4, mu=0.0):
        L = _orc_lib()
        e = _OrcError()
        if case is not None:
            self.h = L.orc_setup(case.encode(), n, degree, int(nonuniform), ctypes.byref(e))
        else:
            xs, ys, zs = (np.ascontiguousarray(a, dtype=np.float64) for a in mesh)
            self.h = L.orc_create(len(xs) - 1, len(ys) - 1, len(zs) - 1, _ptr(xs), _ptr(ys), _ptr(zs),
                                  degree, dim, gamma, mu, ctypes.byref(e))
        if not self.h:
            _raise(e)
        self.L = L
        self.N = L.orc_N(self.h)
        self.ncells = L.orc_ncells(self.h)
        self.ncoeffs = L.orc_ncoeffs(self.h)
        self.degree = degree

    def __del__(self):
        if getattr(self, "h", None):
            self.L.orc_free(self.h)
            self.h = None

    @property
    def state(self) -> np.ndarray:
        p = self.L.orc_state(self.h)
        return np.ctypeslib.as_array(p, shape=(self.ncoeffs,))

    def set_state(self, q):
        self.state[:] = np.asarray(q, dtype=np.float64).ravel()

    def face_npts(self, axis):
        return self.L.orc_face_npts(self.h, axis)

    def residual(self, dt, coeffs=None, faces=False, count=False):
        R = np.zeros(self.ncoeffs)
        Rt = np.zeros(self.ncoeffs)
        fb = [np.zeros(self.ncells * self.face_npts(a) * 10) for a in range(3)] if faces else [None] * 3
        cnt = ctypes.c_long(0)
        e = _OrcError()
        c = None if coeffs is None else np.ascontiguousarray(coeffs, dtype=np.float64)
        rc = self.L.orc_residual(self.h, _ptr(c), dt, _ptr(R), _ptr(Rt), *(_ptr(f) for f in fb),
                                 ctypes.byref(cnt) if count else None, ctypes.byref(e))
        if rc:
            _raise(e)
        out = {"R": R, "Rt": Rt}
        if faces:
            out["faces"] = fb
        if count:
            out["flux_evaluations"] = cnt.value
        return out

    def apply_inverse_mass(self, R):
        R = np.ascontiguousarray(R, dtype=np.float64)
        L = np.empty_like(R)
        self.L.orc_apply_inverse_mass(self.h, _ptr(R), _ptr(L))
        return L

    def compute_dt(self, cfl):
        dt = ctypes.c_double()
        e = _OrcError()
        if self.L.orc_compute_dt(self.h, cfl, ctypes.byref(dt), ctypes.byref(e)):
            _raise(e)
        return dt.value

    def step(self, dt):
        e = _OrcError()
        if self.L.orc_step(self.h, dt, ctypes.byref(e)):
            _raise(e)

    def tgv_diagnostics(self):
        out = np.zeros(2)
        self.L.orc_tgv_diagnostics(self.h, _ptr(out))
        return out

    def error_norms(self, t):
        out = np.zeros(3)
        if self.L.orc_error_norms(self.h, t, _ptr(out)):
            raise OracleError(4, -1, 0.0, "case has no exact solution")
        return out


def orc_interface_flux(tl, tr, gamma, tau, dt):
    L = _orc_lib()
    tl = np.ascontiguousarray(tl, dtype=np.float64)
    tr = np.ascontiguousarray(tr, dtype=np.float64)
    full, half = np.zeros(5), np.zeros(5)
    e = _OrcError()
    if L.orc_interface_flux(_ptr(tl), _ptr(tr), gamma, tau, dt, _ptr(full), _ptr(half), ctypes.byref(e)):
        _raise(e)
    return full, half


def orc_smooth_flux(t, gamma, tau, dt, axis):
    L = _orc_lib()
    t = np.ascontiguousarray(t, dtype=np.float64)
    full, half = np.zeros(5), np.zeros(5)
    e = _OrcError()
    if L.orc_smooth_flux(_ptr(t), gamma, tau, dt, axis, _ptr(full), _ptr(half), ctypes.byref(e)):
        _raise(e)
    return full, half


def orc_moments(prim, gamma):
    L = _orc_lib()
    prim = np.ascontiguousarray(prim, dtype=np.float64)
    out = np.zeros(47)
    L.orc_maxwellian_moments(_ptr(prim), gamma, _ptr(out))
    return out


# --------------------------------------------------------------- reference
_ref = {}


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def native_ref_usable() -> bool:
    """True if the -march=native reference build loads and steps on THIS
    host's CPU (probed in a subprocess: an unsupported ISA would SIGILL)."""
    if not os.path.exists(REF_NATIVE_SO):
        return False
    code = ("import sys; sys.path.insert(0, %r); import oracle as O; "
            "r = O.RefRun('adv3d', 4, 2, lib='native'); r.step(r.compute_dt(0.15))" % os.path.dirname(HERE))
    try:
        return subprocess.run([sys.executable, "-c", code], capture_output=True, timeout=120).returncode == 0
    except (OSError, subprocess.TimeoutExpired):
        return False


def _ref_lib(lib: str = "portable"):
    if lib not in _ref:
        path = {"native": REF_NATIVE_SO, "nofma": REF_NOFMA_SO}.get(lib, REF_SO)
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (needs /root/reference at build time)")
        L = ctypes.CDLL(path)
        L.ref_setup.restype = ctypes.c_void_p
        L.ref_setup.argtypes = [ctypes.c_char_p] + [ctypes.c_int] * 4 + [ctypes.c_char_p, ctypes.c_int]
        L.ref_free.argtypes = [ctypes.c_void_p]
        L.ref_info.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), _dp]
        L.ref_nodes.argtypes = [ctypes.c_void_p, _dp, _dp, _dp]
        L.ref_ncoeffs.restype = ctypes.c_long
        L.ref_ncoeffs.argtypes = [ctypes.c_void_p]
        L.ref_get_state.argtypes = [ctypes.c_void_p, _dp, _dp]
        L.ref_set_state.argtypes = [ctypes.c_void_p, _dp, ctypes.c_double]
        L.ref_residual.argtypes = [ctypes.c_void_p, _dp, ctypes.c_double, ctypes.c_int, _dp, _dp, _dp,
                                   _dp, _dp, ctypes.POINTER(ctypes.c_long), ctypes.c_char_p, ctypes.c_int]
        L.ref_apply_inverse_mass.argtypes = [ctypes.c_void_p, _dp, _dp, ctypes.c_int]
        L.ref_compute_dt.argtypes = [ctypes.c_void_p, ctypes.c_double, _dp, ctypes.c_char_p, ctypes.c_int]
        L.ref_step.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_char_p, ctypes.c_int]
        L.ref_advance.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                  ctypes.c_double, ctypes.c_int, ctypes.POINTER(ctypes.c_int), _dp,
                                  ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_char_p, ctypes.c_int]
        L.ref_tgv_diagnostics.argtypes = [ctypes.c_void_p, _dp]
        L.ref_error_norms.argtypes = [ctypes.c_void_p, ctypes.c_double, _dp, ctypes.c_char_p, ctypes.c_int]
        L.ref_interface_flux.argtypes = [_dp, _dp, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                         _dp, _dp, ctypes.c_char_p, ctypes.c_int]
        L.ref_smooth_flux.argtypes = [_dp, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                      _dp, _dp, ctypes.c_char_p, ctypes.c_int]
        L.ref_maxwellian_moments.argtypes = [_dp, ctypes.c_double, _dp]
        L.ref_tables.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp, _dp, _dp]
        _ref[lib] = L
    return _ref[lib]


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class RefRun:
    """The reference itself (setup_run + residual / step / advance)."""

    def __init__(self, case, n, degree=2, nonuniform=False, workers=1, lib="portable"):
        L = _ref_lib(lib)
        err = ctypes.create_string_buffer(512)
        self.h = L.ref_setup(case.encode(), n, degree, int(nonuniform), workers, err, 512)
        if not self.h:
            raise RefError(2, err.value.decode())
        self.L = L
        dims = (ctypes.c_int * 6)()
        gas = (ctypes.c_double * 3)()
        L.ref_info(self.h, dims, gas)
        self.nx, self.ny, self.nz, self.N, self.dim, self.degree = list(dims)
        self.gamma, self.K, self.mu = list(gas)
        self.ncells = self.nx * self.ny * self.nz
        self.ncoeffs = L.ref_ncoeffs(self.h)
        self.workers = workers
        self.case = case

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_free(self.h)
            self.h = None

    def nodes(self):
        xs, ys, zs = np.zeros(self.nx + 1), np.zeros(self.ny + 1), np.zeros(self.nz + 1)
        self.L.ref_nodes(self.h, _ptr(xs), _ptr(ys), _ptr(zs))
        return xs, ys, zs

    def get_state(self):
        q = np.zeros(self.ncoeffs)
        t = ctypes.c_double()
        self.L.ref_get_state(self.h, _ptr(q), ctypes.byref(t))
        return q, t.value

    def set_state(self, q, t=0.0):
        q = np.ascontiguousarray(q, dtype=np.float64)
        self.L.ref_set_state(self.h, _ptr(q), t)

    def residual(self, dt, coeffs=None, faces=False, count=False, workers=None):
        nq = 3 if self.degree == 3 else 2
        npts = [nq * nq] * 3 if self.dim == 3 else [nq, nq, nq * nq]  # dg.hpp:111-126
        R, Rt = np.zeros(self.ncoeffs), np.zeros(self.ncoeffs)
        fb = [np.zeros(self.ncells * npts[a] * 10) for a in range(3)] if faces else [None] * 3
        cnt = ctypes.c_long(0)
        err = ctypes.create_string_buffer(512)
        c = None if coeffs is None else np.ascontiguousarray(coeffs, dtype=np.float64)
        rc = self.L.ref_residual(self.h, _ptr(c), dt, workers or self.workers, _ptr(R), _ptr(Rt),
                                 *(_ptr(f) for f in fb), ctypes.byref(cnt) if count else None, err, 512)
        if rc:
            raise RefError(rc, err.value.decode())
        out = {"R": R, "Rt": Rt}
        if faces:
            out["faces"] = fb
        if count:
            out["flux_evaluations"] = cnt.value
        return out

    def apply_inverse_mass(self, R):
        R = np.ascontiguousarray(R, dtype=np.float64)
        L = np.empty_like(R)
        self.L.ref_apply_inverse_mass(self.h, _ptr(R), _ptr(L), self.workers)
        return L

    def compute_dt(self, cfl):
        dt = ctypes.c_double()
        err = ctypes.create_string_buffer(512)
        rc = self.L.ref_compute_dt(self.h, cfl, ctypes.byref(dt), err, 512)
        if rc:
            raise RefError(rc, err.value.decode())
        return dt.value

    def step(self, dt, workers=None):
        err = ctypes.create_string_buffer(512)
        rc = self.L.ref_step(self.h, dt, workers or self.workers, err, 512)
        if rc:
            raise RefError(rc, err.value.decode())

    def advance(self, t_end, cfl=0.0, dt_fixed=0.0, record_interval=0.05, workers=None, max_rec=10000):
        steps, nrec = ctypes.c_int(), ctypes.c_int()
        rec = np.zeros(4 * max_rec)
        err = ctypes.create_string_buffer(512)
        rc = self.L.ref_advance(self.h, t_end, cfl, dt_fixed, record_interval, workers or self.workers,
                                ctypes.byref(steps), _ptr(rec), max_rec, ctypes.byref(nrec), err, 512)
        if rc:
            raise RefError(rc, err.value.decode())
        return steps.value, rec[: 4 * nrec.value].reshape(-1, 4)

    def tgv_diagnostics(self):
        out = np.zeros(3)
        self.L.ref_tgv_diagnostics(self.h, _ptr(out))
        return out

    def error_norms(self, t):
        out = np.zeros(3)
        err = ctypes.create_string_buffer(512)
        rc = self.L.ref_error_norms(self.h, t, _ptr(out), err, 512)
        if rc:
            raise RefError(rc, err.value.decode())
        return out


def ref_interface_flux(tl, tr, gamma, tau, dt):
    L = _ref_lib()
    tl = np.ascontiguousarray(tl, dtype=np.float64)
    tr = np.ascontiguousarray(tr, dtype=np.float64)
    full, half = np.zeros(5), np.zeros(5)
    err = ctypes.create_string_buffer(512)
    rc = L.ref_interface_flux(_ptr(tl), _ptr(tr), gamma, tau, dt, _ptr(full), _ptr(half), err, 512)
    if rc:
        raise RefError(rc, err.value.decode())
    return full, half


def ref_smooth_flux(t, gamma, tau, dt, axis):
    L = _ref_lib()
    t = np.ascontiguousarray(t, dtype=np.float64)
    full, half = np.zeros(5), np.zeros(5)
    err = ctypes.create_string_buffer(512)
    rc = L.ref_smooth_flux(_ptr(t), gamma, tau, dt, axis, _ptr(full), _ptr(half), err, 512)
    if rc:
        raise RefError(rc, err.value.decode())
    return full, half


def ref_moments(prim, gamma):
    L = _ref_lib()
    prim = np.ascontiguousarray(prim, dtype=np.float64)
    out = np.zeros(47)
    L.ref_maxwellian_moments(_ptr(prim), gamma, _ptr(out))
    return out


def ref_tables(degree, dim, which):
    L = _ref_lib()
    N = {(1, 3): 4, (2, 3): 10, (3, 3): 20, (2, 2): 6, (3, 2): 10}[(degree, dim)]
    B = np.zeros(125 * N)
    dB = np.zeros(125 * 3 * N)
    w = np.zeros(125)
    ref = np.zeros(125 * 3)
    npts = L.ref_tables(degree, dim, which, _ptr(B), _ptr(dB), _ptr(w), _ptr(ref))
    return B[: npts * N].reshape(npts, N), dB[: npts * 3 * N].reshape(npts, 3, N), w[:npts], ref[: 3 * npts].reshape(npts, 3)


def rel_linf(a, b) -> float:
    """Norm-relative L-inf: max|a-b| / max|b| (SURVEY §8c parity metric)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.max(np.abs(b))
    return float(np.max(np.abs(a - b)) / (den if den > 0 else 1.0))
