"""B200-native DG-HGKS time step (arXiv 2202.13821).

The hot path — kinetic face fluxes, fused volume/projection/inverse-mass/S2O4
cell update — runs in hand-written sm_100a CUDA kernels (csrc/) behind the C
ABI in include/hgks_b200.h. This package is the host-side mirror of the
reference's hgks:: interface over that ABI (see solver.py).
"""
from .solver import (  # noqa: F401
    CaseConfig, ConfigError, CudaError, GasModel, HgksError, InvalidStateError, Mesh,
    NonPositiveDtError, RunOptions, RunResult, Scheme, Solver, TgvRecord, advance, build_mesh,
    case_axis_nodes, compute_dt, default_cfl, dissipation_from_series, residual, run_case,
    setup_run, tgv_record, two_stage_step,
)

__all__ = [
    "CaseConfig", "ConfigError", "CudaError", "GasModel", "HgksError", "InvalidStateError", "Mesh",
    "NonPositiveDtError", "RunOptions", "RunResult", "Scheme", "Solver", "TgvRecord", "advance",
    "build_mesh", "case_axis_nodes", "compute_dt", "default_cfl", "dissipation_from_series",
    "residual", "run_case", "setup_run", "tgv_record", "two_stage_step",
]
