"""Driver layer on the device path: convergence_study and
scaling_report run through the CUDA solver, and the CSV writers format their
results in the reference's layouts (the byte-level format is pinned against
the reference's writers in tests/test_io.py; the norm values against the
reference in tests/test_gpu_acceptance.py)."""
import io

import numpy as np
import pytest

import paper_2202_13821_b200 as P
from paper_2202_13821_b200 import io as hio
from paper_2202_13821_b200.solver import StudyOptions, convergence_study

pytestmark = pytest.mark.gpu


def test_convergence_table_csv(hgks):
    rows = convergence_study("adv2d", [8, 16], StudyOptions(degree=2))
    table = hio.make_error_table([r.n for r in rows], [r.err for r in rows])
    s = io.StringIO()
    hio.write_errors_csv(s, table)
    lines = s.getvalue().splitlines()
    assert lines[0] == "mesh,eL1,orderL1,eL2,orderL2,ec,orderc"
    assert lines[1].startswith("8,") and lines[1].endswith(",")
    assert table[1].order_l1 > 2.0 and table[1].order_l2 > 2.0


def test_scaling_report_and_state_writers(hgks):
    rows = hio.scaling_report("adv3d", [8], [1, 2], degree=2, t_end=0.01)
    assert [r.workers for r in rows] == [1, 2] and rows[0].speedup == 1.0
    s = io.StringIO()
    hio.write_scaling_csv(s, rows)
    assert s.getvalue().startswith("size,workers,seconds,speedup\n8,1,")
    cfg = P.CaseConfig.named("adv3d", 6)
    r = P.run_case(cfg, P.RunOptions(degree=2, t_end=0.01))
    q = r.solver.get_state()[0]
    f, c = io.StringIO(), io.StringIO()
    hio.write_fields_csv(f, q, r.mesh, r.solver.N, cfg.gamma)
    hio.write_coeffs_csv(c, q, r.mesh.ncells(), r.solver.N)
    assert len(f.getvalue().splitlines()) == 1 + 6 ** 3
    assert len(c.getvalue().splitlines()) == 1 + 6 ** 3 * 10
    back = np.array([[float(v) for v in ln.split(",")[2:]] for ln in c.getvalue().splitlines()[1:]])
    assert np.array_equal(back.reshape(-1), np.asarray(q).reshape(-1))  # %.17g round-trips
