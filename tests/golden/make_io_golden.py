"""Golden CSV files from the REFERENCE's writers (io.hpp) for tests/test_io.py.

Writes tests/golden/io/input.txt (the numbers, %.17g) and the five CSVs the
reference writes from them. Compiled without FMA contraction (the oracle's
convention), so the arithmetic inside write_fields_csv is the plain IEEE
sequence the Python mirror performs.

    python tests/golden/make_io_golden.py
"""
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "io")
REF_INC = "/root/reference/proj/include"


def inputs():
    rng = np.random.default_rng(20220228)
    meshes = [8, 16, 32, 64]
    errs = [(3.1e-3 / 8 ** k, 4.7e-3 / 8 ** k, 1.2e-5 / 32 ** k) for k in range(4)]
    recs = [(0.05 * i, 0.125 - 1e-4 * i * i, 4.6875e-4 + 1e-6 * i, 4.6875e-4 * (1 + 0.01 * i)) for i in range(6)]
    rows = [(32, 1, 1.5, 1.0), (32, 4, 0.41, 1.5 / 0.41), (64, 1, 12.25, 1.0), (64, 8, 1.7, 12.25 / 1.7)]
    nx, ny, nz, N, gamma = 3, 2, 2, 10, 1.4
    xi = np.linspace(0.0, 2.0, nx + 1)
    xs = xi + 0.05 * np.sin(np.pi * xi)
    ys = np.linspace(-np.pi, np.pi, ny + 1)
    zs = np.array([0.0, 0.7, 2.0])
    q = rng.normal(size=(nx * ny * nz, N, 5)) * 0.1
    q[:, 0, 0] = 1.0 + 0.2 * rng.random(nx * ny * nz)
    q[:, 0, 4] = 2.5 + rng.random(nx * ny * nz)
    return meshes, errs, recs, rows, (nx, ny, nz, N, gamma), xs, ys, zs, q


def main():
    os.makedirs(OUT, exist_ok=True)
    meshes, errs, recs, rows, dims, xs, ys, zs, q = inputs()
    f = lambda v: "%.17g" % v  # noqa: E731
    lines = [str(len(meshes))] + [f"{n} {f(a)} {f(b)} {f(c)}" for n, (a, b, c) in zip(meshes, errs)]
    lines += [str(len(recs))] + [" ".join(f(v) for v in r) for r in recs]
    lines += [str(len(rows))] + [f"{r[0]} {r[1]} {f(r[2])} {f(r[3])}" for r in rows]
    lines += [" ".join(str(v) for v in dims[:4]) + " " + f(dims[4])]
    lines += [" ".join(f(v) for v in a) for a in (xs, ys, zs)]
    lines += [" ".join(f(v) for v in q.reshape(-1))]
    inp = os.path.join(OUT, "input.txt")
    open(inp, "w").write("\n".join(lines) + "\n")
    exe = "/tmp/hgks_io_driver"
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I" + REF_INC,
                           os.path.join(HERE, "io_driver.cpp"), "-o", exe, "-pthread"])
    subprocess.check_call([exe, inp, OUT])
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    sys.exit(main())
