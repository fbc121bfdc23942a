"""Result tables and CSV writers of the reference's drivers.

Mirrors proj/include/hgks/io.hpp:17-21 (fmt17), :147-215 (ErrorRow,
make_error_table, write_errors_csv / write_tgv_csv / write_scaling_csv /
write_fields_csv / write_coeffs_csv) and solver.hpp:204-229 (scaling_report),
so the files a device run writes are byte-for-byte the files the reference
writes for the same numbers (tests/test_io.py pins this against the
reference's own writers). The numbers come from the device path
(solver.Solver); nothing here computes on the host beyond formatting.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass
from typing import IO, List, Optional, Sequence

import numpy as np


def fmt17(v: float) -> str:
    """io.hpp:17-21: snprintf("%.17g")."""
    return "%.17g" % v


@dataclass
class ErrorRow:
    """io.hpp:147-152: one accuracy-table row; orders empty on the first row."""
    n: int
    e: object  # solver.ErrorNorms
    order_l1: Optional[float] = None
    order_l2: Optional[float] = None
    order_c: Optional[float] = None


def make_error_table(meshes: Sequence[int], errs: Sequence[object]) -> List[ErrorRow]:
    """io.hpp:154-168: orders log2(e_coarse / e_fine) between consecutive meshes."""
    rows = []
    for i, (n, e) in enumerate(zip(meshes, errs)):
        r = ErrorRow(n, e)
        if i > 0:
            p = errs[i - 1]
            r.order_l1 = math.log2(p.l1 / e.l1)
            r.order_l2 = math.log2(p.l2 / e.l2)
            r.order_c = math.log2(p.cell_avg / e.cell_avg)
        rows.append(r)
    return rows


def write_errors_csv(os: IO[str], rows: Sequence[ErrorRow]) -> None:
    """io.hpp:170-175."""
    opt = lambda v: fmt17(v) if v is not None else ""  # noqa: E731
    os.write("mesh,eL1,orderL1,eL2,orderL2,ec,orderc\n")
    for r in rows:
        os.write(f"{r.n},{fmt17(r.e.l1)},{opt(r.order_l1)},{fmt17(r.e.l2)},{opt(r.order_l2)},"
                 f"{fmt17(r.e.cell_avg)},{opt(r.order_c)}\n")


def write_tgv_csv(os: IO[str], recs: Sequence[object]) -> None:
    """io.hpp:177-182 (records: solver.TgvRecord)."""
    os.write("t,Ek,epsEk,epsZeta\n")
    for r in recs:
        os.write(f"{fmt17(r.t)},{fmt17(r.Ek)},{fmt17(r.epsEk)},{fmt17(r.epsZeta)}\n")


@dataclass
class ScalingRow:
    """runtime.hpp:102-107."""
    size: int
    workers: int
    seconds: float
    speedup: float


def write_scaling_csv(os: IO[str], rows: Sequence[ScalingRow]) -> None:
    """io.hpp:184-189."""
    os.write("size,workers,seconds,speedup\n")
    for r in rows:
        os.write(f"{r.size},{r.workers},{fmt17(r.seconds)},{fmt17(r.speedup)}\n")


def _cell_prims(q: np.ndarray, gamma: float):
    """primitive_from_conserved + pressure(Primitive) (core.hpp:72-91) on the
    cell means, in the reference's operation order (so %.17g agrees)."""
    rho, mx, my, mz, E = (q[:, v] for v in range(5))
    p1 = (gamma - 1.0) * (E - 0.5 * (mx * mx + my * my + mz * mz) / rho)
    if np.any(~(rho > 0.0)):
        raise ValueError("non-positive density in write_fields_csv")
    if np.any(~(p1 > 0.0)):
        raise ValueError("non-positive pressure in write_fields_csv")
    inv = 1.0 / rho
    lam = 0.5 * rho / p1
    return rho, mx * inv, my * inv, mz * inv, 0.5 * rho / lam


def write_fields_csv(os: IO[str], coeffs: np.ndarray, mesh, N: int, gamma: float) -> None:
    """io.hpp:192-206: cell-average primitive field (coeffs: AoS [(c*N+n)*5+v])."""
    nc = mesh.ncells()
    q = np.asarray(coeffs, dtype=np.float64).reshape(nc, N, 5)[:, 0, :]
    rho, U, V, W, p = _cell_prims(q, gamma)
    xs, ys, zs = (np.asarray(a, dtype=np.float64) for a in (mesh.xs, mesh.ys, mesh.zs))
    nx, ny = len(xs) - 1, len(ys) - 1
    os.write("i,j,k,x,y,z,rho,u,v,w,p\n")
    for c in range(nc):
        i, j, k = c % nx, (c // nx) % ny, c // (nx * ny)
        xc = 0.5 * (xs[i] + xs[i + 1])
        yc = 0.5 * (ys[j] + ys[j + 1])
        zc = 0.5 * (zs[k] + zs[k + 1])
        os.write(f"{i},{j},{k},{fmt17(xc)},{fmt17(yc)},{fmt17(zc)},{fmt17(rho[c])},{fmt17(U[c])},"
                 f"{fmt17(V[c])},{fmt17(W[c])},{fmt17(p[c])}\n")


def write_coeffs_csv(os: IO[str], coeffs: np.ndarray, ncells: int, N: int) -> None:
    """io.hpp:208-215: every modal coefficient, one (cell, n) per row."""
    q = np.asarray(coeffs, dtype=np.float64).reshape(ncells, N, 5)
    os.write("cell,n,rho,mx,my,mz,E\n")
    for c in range(ncells):
        for n in range(N):
            os.write(f"{c},{n}," + ",".join(fmt17(v) for v in q[c, n]) + "\n")


def scaling_report(case_name: str, sizes: Sequence[int], workers: Sequence[int], degree: int,
                   t_end: Optional[float] = None, device: int = 0) -> List[ScalingRow]:
    """solver.hpp:204-229: wall time of advance() per (size, workers),
    speedup = time(first entry) / time. On the device the worker count does
    not change the computation (results are bitwise independent of it, as in
    the reference), so the rows time identical device runs; the GPU-count
    scaling is bench.py's torchrun path."""
    from .solver import CaseConfig, RunOptions, advance, setup_run

    rows = []
    for n in sizes:
        base = 0.0
        for w in workers:
            cfg = CaseConfig.named(case_name, n)
            opt = RunOptions(degree=degree, workers=w, t_end=t_end, device=device)
            r = setup_run(cfg, opt)
            r.solver.synchronize()
            start = time.perf_counter()
            advance(r, cfg, opt, lambda rr: None)
            r.solver.synchronize()
            secs = time.perf_counter() - start
            r.solver.close()
            if w == 1 or base == 0.0:
                base = secs
            rows.append(ScalingRow(n, w, secs, base / secs))
    return rows
