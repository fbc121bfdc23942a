"""Host-side mirror of the reference solver interface (proj/include/hgks),
driving the B200 kernels through the C ABI (include/hgks_b200.h).

Names, argument meanings and error behaviour follow the reference:

=====================================  =====================================
reference (C++)                        here
=====================================  =====================================
GasModel::make (core.hpp:35)           GasModel.make
Mesh::make (mesh.hpp:22)               Mesh.make
Scheme::make (dg.hpp:274)              Scheme.make
CaseConfig::named (cases.hpp:12)       CaseConfig.named
build_mesh (cases.hpp:59)              build_mesh
setup_run (solver.hpp:29)              setup_run
residual (dg.hpp:354)                  Solver.residual / residual()
apply_inverse_mass (solver.hpp:42)     Solver.apply_inverse_mass
compute_dt (integrator.hpp:27)         Solver.compute_dt / compute_dt()
two_stage_step (integrator.hpp:64)     Solver.step / two_stage_step()
advance (solver.hpp:62)                advance
run_case (solver.hpp:110)              run_case
tgv_diagnostics (cases.hpp:165)        Solver.tgv_diagnostics
project(field, ...) (dg.hpp:193)       Solver.project_field / project_case
error_norms (dg.hpp:228)               Solver.error_norms_field / run_error_norms
dissipation_from_series (:208)         dissipation_from_series
invalid_state_error (core.hpp:58)      InvalidStateError (+ .item/.phase)
non_positive_dt (integrator.hpp:17)    NonPositiveDtError
std::invalid_argument                  ConfigError
=====================================  =====================================

All arithmetic runs in the CUDA library; this module only moves host
arrays across the ABI.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _lib
from ._lib import HgksConfig

_dp = ctypes.POINTER(ctypes.c_double)


# ------------------------------------------------------------------- errors
class HgksError(RuntimeError):
    pass


class InvalidStateError(HgksError):
    """invalid_state_error: non-positive density or pressure (core.hpp:58-70),
    message shaped like worker_error (runtime.hpp:37-41)."""

    def __init__(self, msg, item=-1, phase=-1, value=0.0):
        super().__init__(msg)
        self.item, self.phase, self.value = item, phase, value


class NonPositiveDtError(HgksError):
    """non_positive_dt (integrator.hpp:17-19)."""


class ConfigError(HgksError, ValueError):
    """configuration error (std::invalid_argument in the reference)."""


class CudaError(HgksError):
    pass


def _raise(L, h, rc):
    msg = L.hgks_last_error(h).decode() if h else "hgks error"
    if rc == _lib.HGKS_ERR_STATE:
        code, phase, item, val = ctypes.c_int(), ctypes.c_int(), ctypes.c_long(), ctypes.c_double()
        L.hgks_error_info(h, ctypes.byref(code), ctypes.byref(phase), ctypes.byref(item), ctypes.byref(val))
        raise InvalidStateError(msg, item.value, phase.value, val.value)
    if rc == _lib.HGKS_ERR_DT:
        raise NonPositiveDtError(msg)
    if rc == _lib.HGKS_ERR_CONFIG:
        raise ConfigError(msg)
    raise CudaError(msg)


def _ptr(a):
    if a is None:
        return None
    if not (a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]):
        raise TypeError("expected a C-contiguous float64 array")
    return a.ctypes.data_as(_dp)


# ------------------------------------------------------- gas, mesh, scheme
@dataclass
class GasModel:
    """core.hpp:29-43. K = (5 - 3 gamma)/(gamma - 1); mu_ref = 0 is Euler."""
    gamma: float
    K: float
    Pr: float = 1.0
    mu_ref: float = 0.0

    @staticmethod
    def make(gamma: float, mu: float = 0.0) -> "GasModel":
        K = (5.0 - 3.0 * gamma) / (gamma - 1.0)
        if K < 0.0:
            raise ConfigError("GasModel: gamma gives negative internal dof")
        return GasModel(gamma=gamma, K=K, mu_ref=mu)


@dataclass
class Mesh:
    """mesh.hpp:11-64: periodic box, per-axis node arrays, x fastest."""
    xs: np.ndarray
    ys: np.ndarray
    zs: np.ndarray

    @staticmethod
    def make(xs, ys, zs) -> "Mesh":
        xs, ys, zs = (np.ascontiguousarray(a, dtype=np.float64) for a in (xs, ys, zs))
        for a in (xs, ys, zs):
            if len(a) < 2 or np.any(np.diff(a) <= 0):
                raise ConfigError("Mesh: node coordinates must be strictly increasing")
        return Mesh(xs, ys, zs)

    @property
    def nx(self):
        return len(self.xs) - 1

    @property
    def ny(self):
        return len(self.ys) - 1

    @property
    def nz(self):
        return len(self.zs) - 1

    def ncells(self) -> int:
        return self.nx * self.ny * self.nz

    def cell_index(self, i, j, k):
        return i + self.nx * (j + self.ny * k)

    def widths(self, c):
        i, j, k = c % self.nx, (c // self.nx) % self.ny, c // (self.nx * self.ny)
        return (self.xs[i + 1] - self.xs[i], self.ys[j + 1] - self.ys[j], self.zs[k + 1] - self.zs[k])

    def volume(self, c):
        h = self.widths(c)
        return h[0] * h[1] * h[2]


def basis_size(degree: int, dim: int) -> int:
    """BasisSet::N for total degree <= k (basis.hpp:64-82)."""
    return sum(1 for a in range(degree + 1) for b in range(degree + 1)
               for c in range(degree + 1 if dim == 3 else 1) if a + b + c <= degree)


@dataclass
class Scheme:
    """dg.hpp:269-281 (the tables live on the device inside Solver)."""
    degree: int
    dim: int
    gas: GasModel
    N: int = 0

    @staticmethod
    def make(degree: int, dim: int, gas: GasModel) -> "Scheme":
        if degree not in (1, 2, 3):
            raise ConfigError("build_basis: degree must be 2 or 3 (1 = P1 extension)")
        if dim not in (2, 3):
            raise ConfigError("build_basis: dim must be 2 or 3")
        return Scheme(degree, dim, gas, basis_size(degree, dim))


def default_cfl(degree: int) -> float:
    """integrator.hpp:22 (0.15 for P2, 0.09 otherwise). P1 (extension, unpinned)
    keeps the reference's formula."""
    return 0.15 if degree == 2 else 0.09


# ------------------------------------------------------------------ solver
class Solver:
    """One device-resident DG-HGKS discretisation (mesh + scheme + state),
    the object behind every call the reference makes per step."""

    def __init__(self, mesh: Mesh, scheme: Scheme, device: int = 0, z_begin: int = 0,
                 z_count: int = 0):
        L = _lib.load()
        self.L = L
        self.mesh, self.scheme = mesh, scheme
        self._keep = (mesh.xs, mesh.ys, mesh.zs)
        cfg = HgksConfig(mesh.nx, mesh.ny, mesh.nz, _ptr(mesh.xs), _ptr(mesh.ys), _ptr(mesh.zs),
                         scheme.degree, scheme.dim, scheme.gas.gamma, scheme.gas.mu_ref, device,
                         z_begin, z_count)
        h = ctypes.c_void_p()
        rc = L.hgks_create(ctypes.byref(cfg), ctypes.byref(h))
        self.h = h.value
        if rc != 0:
            try:
                _raise(L, self.h, rc)
            finally:
                if self.h:
                    L.hgks_destroy(self.h)
                    self.h = None
        self.N = L.hgks_num_basis(self.h)
        self.ncoeffs = L.hgks_num_coeffs(self.h)
        self.z_begin, self.z_count = z_begin, (z_count if z_count > 0 else mesh.nz)
        self._cbs = []

    def close(self):
        if getattr(self, "h", None):
            self.L.hgks_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def _check(self, rc):
        if rc != 0:
            _raise(self.L, self.h, rc)

    def face_points(self, axis: int) -> int:
        return self.L.hgks_face_points(self.h, axis)

    # -- state (DGState, dg.hpp:18-38)
    def set_state(self, coeffs, time: float = 0.0):
        q = np.ascontiguousarray(coeffs, dtype=np.float64).ravel()
        if q.size != self.ncoeffs:
            raise ConfigError(f"state has {q.size} coefficients, expected {self.ncoeffs}")
        self._check(self.L.hgks_set_state(self.h, _ptr(q), time))

    def get_state(self):
        q = np.empty(self.ncoeffs)
        t = ctypes.c_double()
        self._check(self.L.hgks_get_state(self.h, _ptr(q), ctypes.byref(t)))
        return q, t.value

    @property
    def time(self) -> float:
        t = ctypes.c_double()
        self._check(self.L.hgks_get_state(self.h, None, ctypes.byref(t)))
        return t.value

    # -- the hot path
    def residual(self, dt: float, coeffs=None, faces: bool = False):
        """residual() (dg.hpp:354): returns {"R", "Rt"[, "faces"]} in the
        reference layouts (ws.R, ws.Rt, ws.face[a])."""
        R = np.empty(self.ncoeffs)
        Rt = np.empty(self.ncoeffs)
        ncell_owned = self.ncoeffs // (5 * self.N)
        fb = [np.empty(ncell_owned * self.face_points(a) * 10) for a in range(3)] if faces else [None] * 3
        c = None if coeffs is None else np.ascontiguousarray(coeffs, dtype=np.float64).ravel()
        if c is not None and c.size != self.ncoeffs:
            raise ConfigError(f"coeffs has {c.size} values, expected {self.ncoeffs}")
        self._check(self.L.hgks_residual(self.h, _ptr(c), dt, _ptr(R), _ptr(Rt), *(_ptr(f) for f in fb)))
        out = {"R": R, "Rt": Rt}
        if faces:
            out["faces"] = fb
        return out

    def apply_inverse_mass(self, R):
        R = np.ascontiguousarray(R, dtype=np.float64).ravel()
        if R.size != self.ncoeffs:
            raise ConfigError(f"R has {R.size} values, expected {self.ncoeffs}")
        L = np.empty_like(R)
        self._check(self.L.hgks_apply_inverse_mass(self.h, _ptr(R), _ptr(L)))
        return L

    def compute_dt(self, cfl: float) -> float:
        dt = ctypes.c_double()
        self._check(self.L.hgks_compute_dt(self.h, cfl, ctypes.byref(dt)))
        return dt.value

    def step(self, dt: float):
        """two_stage_step on the device-resident state."""
        self._check(self.L.hgks_step(self.h, dt))

    def two_stage_step_host(self, q: np.ndarray, dt: float):
        """two_stage_step(q, dt, eval, scratch) on a host vector, in place."""
        if not (q.dtype == np.float64 and q.flags["C_CONTIGUOUS"] and q.size == self.ncoeffs):
            raise ConfigError("q must be a contiguous float64 vector of the state size")
        self._check(self.L.hgks_two_stage_step_host(self.h, _ptr(q), dt))

    def two_stage_step_host_streamed(self, q: np.ndarray, dt: float, nchunks: int = 0):
        """The host-vector step with H2D / compute / D2H overlapped over z chunks
        (bitwise identical results; on a state error q may be partially advanced)."""
        if not (q.dtype == np.float64 and q.flags["C_CONTIGUOUS"] and q.size == self.ncoeffs):
            raise ConfigError("q must be a contiguous float64 vector of the state size")
        self._check(self.L.hgks_two_stage_step_host_streamed(self.h, _ptr(q), dt, nchunks))

    def advance_to(self, t_end: float, cfl: float, dt_fixed: float = 0.0, record_interval: float = 0.0) -> int:
        n = ctypes.c_int()
        self._check(self.L.hgks_advance(self.h, t_end, cfl, dt_fixed, record_interval, ctypes.byref(n)))
        return n.value

    def advance_records(self, t_end: float, cfl: float, dt_fixed: float = 0.0, record_interval: float = 0.0,
                        first_record: float = 0.0, max_steps: int = 0,
                        on_record: Optional[Callable[[float], None]] = None) -> int:
        """hgks_advance_records: the device-resident loop (dt, clipping, commit
        and failure checks on the GPU, one CUDA graph per step);
        on_record(t) runs after each step that lands on a record time, with
        the solver showing that step's state."""
        n = ctypes.c_int()
        err = []

        def cb(user, h, t):
            try:
                on_record(t)
                return 0
            except Exception as e:  # noqa: BLE001 — re-raised below
                err.append(e)
                return 1
        c = _lib.RECORD_FN(cb) if on_record is not None else _lib.RECORD_FN()
        rc = self.L.hgks_advance_records(self.h, t_end, cfl, dt_fixed, record_interval, first_record,
                                         max_steps, c, None, ctypes.byref(n))
        if err:
            raise err[0]
        self._check(rc)
        return n.value

    # -- cases, diagnostics
    def project_case(self, case_name: str, t: float = 0.0):
        self._check(self.L.hgks_project_case(self.h, case_name.encode(), t))

    def error_norm_sums(self, case_name: str, t: float):
        """Unreduced error_norms sums over owned cells: (L1, L2^2, cell-avg^2)."""
        out = np.zeros(3)
        self._check(self.L.hgks_error_norms(self.h, case_name.encode(), t, _ptr(out)))
        return out

    def error_norms(self, case_name: str, t: float):
        """error_norms (dg.hpp:228-266): (l1, l2, cell_avg) against the exact field."""
        s = self.error_norm_sums(case_name, t)
        return np.array([s[0], np.sqrt(s[1]), np.sqrt(s[2])])

    def projection_points(self) -> np.ndarray:
        """Physical coordinates [cell, p, 3] of the projection points of the
        owned cells: x = center + h/2 * ref_p over the (k+2)^dim Gauss points,
        (i, j, k) order with k fastest (dg.hpp:102-105, :193-220); z is 0 in 2-D."""
        npts = self.L.hgks_projection_npts(self.h)
        dim = self.scheme.dim
        nq = int(round(npts ** (1.0 / dim)))
        g = np.polynomial.legendre.leggauss(nq)[0]
        if dim == 3:
            ref = np.array([(g[a], g[b], g[c]) for a in range(nq) for b in range(nq) for c in range(nq)])
        else:
            ref = np.array([(g[a], g[b], 0.0) for a in range(nq) for b in range(nq)])
        m = self.mesh
        cx, hx = 0.5 * (m.xs[1:] + m.xs[:-1]), np.diff(m.xs)
        cy, hy = 0.5 * (m.ys[1:] + m.ys[:-1]), np.diff(m.ys)
        cz, hz = 0.5 * (m.zs[1:] + m.zs[:-1]), np.diff(m.zs)
        ks = np.arange(self.z_begin, self.z_begin + self.z_count)
        K, J, I = np.meshgrid(ks, np.arange(m.ny), np.arange(m.nx), indexing="ij")
        I, J, K = I.ravel(), J.ravel(), K.ravel()   # owned cells, x fastest
        pts = np.empty((I.size, npts, 3))
        pts[:, :, 0] = cx[I, None] + 0.5 * hx[I, None] * ref[None, :, 0]
        pts[:, :, 1] = cy[J, None] + 0.5 * hy[J, None] * ref[None, :, 1]
        pts[:, :, 2] = cz[K, None] + 0.5 * hz[K, None] * ref[None, :, 2] if dim == 3 else 0.0
        return pts

    def _sample(self, field, rho_only: bool) -> np.ndarray:
        pts = self.projection_points()
        q = np.asarray(field(pts[..., 0], pts[..., 1], pts[..., 2]), dtype=np.float64)
        if q.shape != (5,) + pts.shape[:2]:
            raise ConfigError(f"field must return 5 conserved arrays shaped {pts.shape[:2]}, got {q.shape}")
        return np.ascontiguousarray(q[0] if rho_only else np.moveaxis(q, 0, -1)).ravel()

    def project_field(self, field, t: float = 0.0):
        """project(field, mesh, tab, part) (dg.hpp:193-220) for a caller field:
        field(x, y, z) -> (rho, rho U, rho V, rho W, E) arrays over the
        projection points (numpy broadcasting); the quadrature sums run on the
        device (hgks_project_samples)."""
        smp = self._sample(field, False)
        self._check(self.L.hgks_project_samples(self.h, _ptr(smp), t))

    def error_norms_field(self, exact):
        """error_norms(state, mesh, tab, exact, part) (dg.hpp:228-266) against a
        caller field (its density): unreduced (L1, L2^2, cell-avg^2) sums, as
        error_norm_sums."""
        rho = self._sample(exact, True)
        out = np.zeros(3)
        self._check(self.L.hgks_error_norms_samples(self.h, _ptr(rho), _ptr(out)))
        return out

    def tgv_diagnostics(self):
        """(Ek*vol, enstrophy*vol, vol) sums over owned cells (cases.hpp:165-204)."""
        e, z, v = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        self._check(self.L.hgks_tgv_diagnostics(self.h, ctypes.byref(e), ctypes.byref(z), ctypes.byref(v)))
        return e.value, z.value, v.value

    # -- debug / plumbing
    def set_count_fluxes(self, on: bool = True):
        self.L.hgks_set_count_fluxes(self.h, int(on))

    def flux_evaluations(self) -> int:
        return self.L.hgks_flux_evaluations(self.h)

    def launch_count(self) -> int:
        return self.L.hgks_launch_count(self.h)

    def synchronize(self):
        self._check(self.L.hgks_synchronize(self.h))

    def set_stream(self, stream_ptr: Optional[int]):
        self._check(self.L.hgks_set_stream(self.h, stream_ptr))

    def stream(self) -> int:
        return self.L.hgks_get_stream(self.h) or 0

    def set_kernel_timing(self, on: bool = True):
        self.L.hgks_set_kernel_timing(self.h, int(on))

    def kernel_times(self):
        f, c, o = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        self.L.hgks_kernel_times(self.h, ctypes.byref(f), ctypes.byref(c), ctypes.byref(o))
        return f.value, c.value

    def kernel_times_stage(self, stage: int):
        """(face ms, cell ms) of one S2O4 stage of the last timed step."""
        f, c = ctypes.c_double(), ctypes.c_double()
        self._check(self.L.hgks_kernel_times_stage(self.h, stage, ctypes.byref(f), ctypes.byref(c)))
        return f.value, c.value

    # -- multi-slab plumbing
    def halo_bytes(self) -> int:
        return self.L.hgks_halo_bytes(self.h)

    def halo_buffers(self):
        """device addresses of the packed halo buffers (send_lo, send_hi, recv_lo, recv_hi)."""
        vals = [ctypes.c_ulonglong() for _ in range(4)]
        self._check(self.L.hgks_halo_buffers(self.h, *(ctypes.byref(v) for v in vals)))
        return tuple(v.value for v in vals)

    def halo_pack(self, which: int):
        self._check(self.L.hgks_halo_pack(self.h, which))

    def halo_unpack(self, which: int):
        self._check(self.L.hgks_halo_unpack(self.h, which))

    def step_phase(self, dt: float, phase: int):
        self._check(self.L.hgks_step_phase(self.h, dt, phase))

    def set_halo_exchange(self, fn: Callable[["Solver", int], None]):
        """fn(solver, which) moves send_lo -> lower neighbour recv_hi and
        send_hi -> upper neighbour recv_lo (on the solver's stream)."""
        def cb(user, h, which):
            try:
                fn(self, which)
                return 0
            except Exception:  # noqa: BLE001 — reported as an ABI failure
                import traceback
                traceback.print_exc()
                return 1
        c = _lib.HALO_FN(cb)
        self._cbs.append(c)
        self.L.hgks_set_halo_exchange(self.h, c, None)

    def set_halo_exchange_split(self, start: Callable[["Solver", int], None],
                                finish: Callable[["Solver", int], None]):
        """Overlapped exchange: start(solver, which) enqueues the transfer
        behind the solver stream, the ghost-free faces are launched, then
        finish(solver, which) makes the solver stream wait for it."""
        def wrap(fn):
            def cb(user, h, which):
                try:
                    fn(self, which)
                    return 0
                except Exception:  # noqa: BLE001 — reported as an ABI failure
                    import traceback
                    traceback.print_exc()
                    return 1
            return _lib.HALO_FN(cb)
        a, b = wrap(start), wrap(finish)
        self._cbs += [a, b]
        self.L.hgks_set_halo_exchange_split(self.h, a, b, None)

    def set_host_reduce(self, fn: Callable[[int, np.ndarray], None]):
        """fn(op, values) reduces `values` in place over the slabs: op 0 = min
        of uint64 (error keys, dt bits), op 1 = sum of float64."""
        def cb(user, op, ptr, n):
            try:
                ct = ctypes.c_uint64 if op == _lib.HGKS_REDUCE_MIN_U64 else ctypes.c_double
                arr = np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ct)), shape=(n,))
                fn(op, arr)
                return 0
            except Exception:  # noqa: BLE001 — reported as an ABI failure
                import traceback
                traceback.print_exc()
                return 1
        c = _lib.REDUCE_FN(cb)
        self._cbs.append(c)
        self.L.hgks_set_host_reduce(self.h, c, None)

    # -- in-library NCCL data plane
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        rc = _lib.load().hgks_nccl_unique_id(buf, 128)
        if rc != 0:
            raise CudaError("ncclGetUniqueId failed (libnccl.so.2 not loadable?)")
        return buf.raw

    def attach_nccl(self, unique_id: bytes, rank: int, world: int):
        """Join the z-slab ring: halos, dt and error keys over NCCL inside the
        library (no Python on the step path)."""
        self._check(self.L.hgks_attach_nccl(self.h, unique_id, rank, world))

    def slab_reduce_sum(self, values):
        v = np.ascontiguousarray(values, dtype=np.float64).copy()
        self._check(self.L.hgks_slab_reduce_sum(self.h, _ptr(v), v.size))
        return v

    def set_graphs(self, on: bool = True):
        self.L.hgks_set_graphs(self.h, int(on))

    def set_grid_cap(self, ctas: int):
        """Test hook: cap the persistent grids (every CTA walks many tiles)."""
        self.L.hgks_set_grid_cap(self.h, int(ctas))

    def set_face_tma(self, on: bool = True):
        """Face-kernel staging: TMA boxes (default, even nx) or per-lane cp.async."""
        self.L.hgks_set_face_tma(self.h, int(on))

    def set_cell_tma(self, on: bool = True):
        """Cell-kernel staging: TMA boxes (default, even nx) or per-lane cp.async."""
        self.L.hgks_set_cell_tma(self.h, int(on))

    def set_race_shake(self, seed: int):
        """Test hook: randomized per-warp delays before every cp.async wait and
        barrier of the persistent kernels (0 = off)."""
        self.L.hgks_set_race_shake(self.h, int(seed))


def measure_fp64_peak(device: int = 0, ms: float = 50.0) -> float:
    """Sustained DFMA throughput (TFLOP/s) of the device: the FP64 roofline
    denominator (MEASURED_PEAKS.json has no FP64 entry)."""
    L = _lib.load()
    t = ctypes.c_double()
    rc = L.hgks_measure_fp64_peak(device, ms, ctypes.byref(t))
    if rc != 0:
        raise CudaError("fp64 peak measurement failed")
    return t.value


# --------------------------------------------------------------- the cases
@dataclass
class CaseConfig:
    """cases.hpp:12-46."""
    name: str
    dim: int = 2
    n: int = 8
    nonuniform: bool = False
    gamma: float = 1.4
    mach0: float = 0.1
    reynolds: float = 1600.0
    eps: float = 5.0
    t_end: float = 2.0

    @staticmethod
    def named(name: str, n: int) -> "CaseConfig":
        table = {"adv2d": (2, 2.0), "adv3d": (3, 2.0), "vortex2d": (2, 10.0), "tgv": (3, 10.0)}
        if name not in table:
            raise ConfigError("unknown case: " + name)
        dim, t_end = table[name]
        return CaseConfig(name=name, dim=dim, n=n, t_end=t_end)

    def viscosity(self) -> float:
        return 1.0 / self.reynolds if self.name == "tgv" else 0.0


def case_axis_nodes(lo: float, hi: float, n: int, nonuniform: bool) -> np.ndarray:
    """cases.hpp:50-57: x = xi + 0.05 sin(pi xi) on the uniform parameter nodes."""
    xi = np.array([lo + (hi - lo) * i / n for i in range(n + 1)])
    return xi + 0.05 * np.sin(np.pi * xi) if nonuniform else xi


def build_mesh(cfg: CaseConfig) -> Mesh:
    """cases.hpp:59-73 (2-D cases: one z cell spanning the domain)."""
    if cfg.n < 4:
        raise ConfigError("build_mesh: need at least 4 cells per axis")
    lo, hi = 0.0, 2.0
    if cfg.name == "vortex2d":
        hi = 10.0
    if cfg.name == "tgv":
        lo, hi = -math.pi, math.pi
    ax = case_axis_nodes(lo, hi, cfg.n, cfg.nonuniform)
    if cfg.dim == 2:
        return Mesh.make(ax, ax, np.array([lo, hi]))
    return Mesh.make(ax, ax.copy(), ax.copy())


@dataclass
class RunOptions:
    """solver.hpp:10-17."""
    degree: int = 2
    cfl: float = 0.0
    dt_fixed: Optional[float] = None
    t_end: Optional[float] = None
    workers: int = 1  # accepted for interface parity; the device ignores it
    record_interval: float = 0.05
    device: int = 0


@dataclass
class TgvRecord:
    t: float
    Ek: float
    epsEk: float = 0.0
    epsZeta: float = 0.0


@dataclass
class RunResult:
    mesh: Mesh
    scheme: Scheme
    solver: Solver
    steps: int = 0
    records: List[TgvRecord] = field(default_factory=list)

    @property
    def state(self):
        return self.solver.get_state()[0]


def setup_run(cfg: CaseConfig, opt: RunOptions, z_begin: int = 0, z_count: int = 0) -> RunResult:
    """solver.hpp:29-37: mesh, scheme, projected initial state (on device)."""
    mesh = build_mesh(cfg)
    scheme = Scheme.make(opt.degree, cfg.dim, GasModel.make(cfg.gamma, cfg.viscosity()))
    s = Solver(mesh, scheme, device=opt.device, z_begin=z_begin, z_count=z_count)
    s.project_case(cfg.name, 0.0)
    return RunResult(mesh, scheme, s)


def tgv_record(r: RunResult, reduce: Optional[Callable] = None) -> TgvRecord:
    """tgv_diagnostics (cases.hpp:165-204); `reduce` sums partials over ranks."""
    e, z, v = r.solver.tgv_diagnostics()
    if reduce is not None:
        e, z, v = reduce((e, z, v))
    return TgvRecord(t=r.solver.time, Ek=e / v, epsZeta=2.0 * r.scheme.gas.mu_ref * z / v)


def advance(r: RunResult, cfg: CaseConfig, opt: RunOptions, on_record: Callable[[RunResult], None]):
    """solver.hpp:62-108: dt from compute_dt (or dt_fixed), clipped to t_end and
    the next record; the same full dt drives both residuals; state errors get
    " at t=<t>" appended."""
    cfl = opt.cfl if opt.cfl > 0 else default_cfl(opt.degree)
    t_end = opt.t_end if opt.t_end is not None else cfg.t_end
    record = cfg.name == "tgv"
    next_record = opt.record_interval
    on_record(r)
    dt_fixed = opt.dt_fixed if opt.dt_fixed is not None else 0.0
    # the device-resident loop (hgks_advance_records): dt = compute_dt (or
    # dt_fixed) clipped to t_end and, for tgv, to the next record, exactly as
    # solver.hpp:91-93; on_record runs at each record time; " at t=<t>" is
    # appended to state errors
    r.steps += r.solver.advance_records(t_end, cfl, dt_fixed, opt.record_interval if record else 0.0,
                                        next_record, 0, (lambda t: on_record(r)) if record else None)


def dissipation_from_series(ek, dt):
    """cases.hpp:208-216."""
    n = len(ek)
    if n < 3:
        raise ConfigError("dissipation_from_series: need at least 3 samples")
    eps = [0.0] * n
    eps[0] = -(-3.0 * ek[0] + 4.0 * ek[1] - ek[2]) / (2.0 * dt)
    for i in range(1, n - 1):
        eps[i] = -(ek[i + 1] - ek[i - 1]) / (2.0 * dt)
    eps[n - 1] = -(3.0 * ek[n - 1] - 4.0 * ek[n - 2] + ek[n - 3]) / (2.0 * dt)
    return eps


def run_case(cfg: CaseConfig, opt: RunOptions) -> RunResult:
    """solver.hpp:110-126."""
    r = setup_run(cfg, opt)

    def rec(rr):
        if cfg.name == "tgv":
            rr.records.append(tgv_record(rr))

    advance(r, cfg, opt, rec)
    if len(r.records) >= 3:
        eps = dissipation_from_series([x.Ek for x in r.records], opt.record_interval)
        for x, e in zip(r.records, eps):
            x.epsEk = e
    return r


@dataclass
class ErrorNorms:
    """dg.hpp:222-224."""
    l1: float
    l2: float
    cell_avg: float


def run_error_norms(r: RunResult, cfg: CaseConfig) -> ErrorNorms:
    """solver.hpp:129-134 (device error_norms, dg.hpp:228-266)."""
    l1, l2, ec = r.solver.error_norms(cfg.name, r.solver.time)
    return ErrorNorms(float(l1), float(l2), float(ec))


@dataclass
class StudyOptions:
    """solver.hpp:143-152."""
    degree: int = 2
    nonuniform: bool = False
    workers: int = 1
    nominal: bool = False
    dt_power: float = 2.0
    dt_safety: float = 0.7
    anchor_index: int = 0
    cfl: Optional[float] = None
    device: int = 0


@dataclass
class StudyRow:
    n: int
    err: ErrorNorms
    steps: int
    dt: float


def convergence_study(case_name: str, meshes: List[int], sopt: StudyOptions) -> List[StudyRow]:
    """solver.hpp:161-202: per mesh run_case + error norms; refined mode uses
    dt = min(anchor_dt (n_anchor/n)^power, cfl_dt(n)), nominal the CFL step."""
    cfl = sopt.cfl if sopt.cfl is not None else default_cfl(sopt.degree)

    def cfl_dt(n):
        cfg = CaseConfig.named(case_name, n)
        cfg.nonuniform = sopt.nonuniform
        r = setup_run(cfg, RunOptions(degree=sopt.degree, device=sopt.device))
        dt = r.solver.compute_dt(cfl)
        r.solver.close()
        return dt

    anchor_dt, anchor_n = 0.0, 0
    if not sopt.nominal:
        anchor_n = meshes[min(sopt.anchor_index, len(meshes) - 1)]
        anchor_dt = sopt.dt_safety * cfl_dt(anchor_n)
    rows = []
    for n in meshes:
        cfg = CaseConfig.named(case_name, n)
        cfg.nonuniform = sopt.nonuniform
        opt = RunOptions(degree=sopt.degree, cfl=cfl, device=sopt.device)
        if not sopt.nominal:
            policy = anchor_dt * (anchor_n / n) ** sopt.dt_power
            opt.dt_fixed = min(policy, cfl_dt(n))
        r = run_case(cfg, opt)
        rows.append(StudyRow(n, run_error_norms(r, cfg), r.steps, opt.dt_fixed or 0.0))
        r.solver.close()
    return rows


def order(coarse: StudyRow, fine: StudyRow, norm: str) -> float:
    return math.log2(getattr(coarse.err, norm) / getattr(fine.err, norm))


# ------------------------------------------------ free-function spellings
def residual(solver: Solver, q, dt: float):
    return solver.residual(dt, coeffs=q)


def compute_dt(solver: Solver, cfl: float) -> float:
    return solver.compute_dt(cfl)


def two_stage_step(q: np.ndarray, dt: float, solver: Solver):
    solver.two_stage_step_host(q, dt)
