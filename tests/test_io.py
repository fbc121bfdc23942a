"""The device-side result writers (paper_2202_13821_b200/io.py) produce the
reference's CSV files byte for byte (io.hpp:147-215): golden files written by
the reference's own writers from tests/golden/io/input.txt
(tests/golden/make_io_golden.py)."""
import io
import os

import numpy as np

from paper_2202_13821_b200 import io as hio
from paper_2202_13821_b200.solver import ErrorNorms, Mesh, TgvRecord

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")


def _inputs():
    tok = open(os.path.join(GOLD, "input.txt")).read().split()
    pos = 0

    def take(n=1):
        nonlocal pos
        out = tok[pos:pos + n]
        pos += n
        return out

    ne = int(take()[0])
    meshes, errs = [], []
    for _ in range(ne):
        n, a, b, c = take(4)
        meshes.append(int(n))
        errs.append(ErrorNorms(float(a), float(b), float(c)))
    recs = [TgvRecord(*map(float, take(4))) for _ in range(int(take()[0]))]
    rows = []
    for _ in range(int(take()[0])):
        s, w, sec, sp = take(4)
        rows.append(hio.ScalingRow(int(s), int(w), float(sec), float(sp)))
    nx, ny, nz, N = map(int, take(4))
    gamma = float(take()[0])
    xs = np.array(take(nx + 1), dtype=np.float64)
    ys = np.array(take(ny + 1), dtype=np.float64)
    zs = np.array(take(nz + 1), dtype=np.float64)
    q = np.array(take(nx * ny * nz * N * 5), dtype=np.float64)
    assert pos == len(tok)
    return meshes, errs, recs, rows, Mesh.make(xs, ys, zs), N, gamma, q


def _gold(name):
    return open(os.path.join(GOLD, name)).read()


def _render(fn, *args):
    s = io.StringIO()
    fn(s, *args)
    return s.getvalue()


def test_errors_csv_bytes():
    meshes, errs, *_ = _inputs()
    assert _render(hio.write_errors_csv, hio.make_error_table(meshes, errs)) == _gold("errors.csv")


def test_tgv_csv_bytes():
    _, _, recs, *_ = _inputs()
    assert _render(hio.write_tgv_csv, recs) == _gold("tgv.csv")


def test_scale_csv_bytes():
    rows = _inputs()[3]
    assert _render(hio.write_scaling_csv, rows) == _gold("scale.csv")


def test_fields_and_coeffs_csv_bytes():
    _, _, _, _, mesh, N, gamma, q = _inputs()
    assert _render(hio.write_fields_csv, q, mesh, N, gamma) == _gold("fields.csv")
    assert _render(hio.write_coeffs_csv, q, mesh.ncells(), N) == _gold("coeffs.csv")


def test_error_table_orders():
    e = [ErrorNorms(8.0, 4.0, 2.0), ErrorNorms(1.0, 1.0, 1.0)]
    rows = hio.make_error_table([8, 16], e)
    assert rows[0].order_l1 is None and rows[1].order_l1 == 3.0 and rows[1].order_l2 == 2.0
    assert rows[1].order_c == 1.0
