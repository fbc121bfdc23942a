"""ctypes binding of include/hgks_b200.h (libhgks_b200.so, built in-tree).

There is no fallback: if the CUDA library is missing or cannot load, import
fails with the reason. Build it with ``python -m paper_2202_13821_b200.build``
(or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# HGKS_LIB selects an alternate build (kernel-variant experiments only)
LIB_PATH = os.environ.get("HGKS_LIB") or os.path.join(HERE, "libhgks_b200.so")

HGKS_OK, HGKS_ERR_STATE, HGKS_ERR_CONFIG, HGKS_ERR_DT, HGKS_ERR_CUDA = 0, 1, 2, 3, 4

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_lp = ctypes.POINTER(ctypes.c_long)
_u64p = ctypes.POINTER(ctypes.c_ulonglong)

# every symbol include/hgks_b200.h declares (tests check the export table)
EXPORTS = [
    "hgks_abi_version", "hgks_create", "hgks_destroy", "hgks_last_error", "hgks_error_info",
    "hgks_num_basis", "hgks_num_coeffs", "hgks_face_points", "hgks_set_state", "hgks_get_state",
    "hgks_residual", "hgks_apply_inverse_mass", "hgks_compute_dt", "hgks_compute_dt_k", "hgks_step",
    "hgks_two_stage_step_host", "hgks_two_stage_step_host_streamed", "hgks_advance_records", "hgks_advance",
    "hgks_set_count_fluxes", "hgks_flux_evaluations",
    "hgks_project_case", "hgks_tgv_diagnostics", "hgks_error_norms", "hgks_projection_npts",
    "hgks_project_samples", "hgks_error_norms_samples", "hgks_halo_bytes", "hgks_halo_buffers",
    "hgks_halo_pack", "hgks_halo_unpack", "hgks_set_halo_exchange", "hgks_set_halo_exchange_split", "hgks_step_phase",
    "hgks_set_host_reduce", "hgks_nccl_unique_id", "hgks_attach_nccl", "hgks_attach_nccl_comm",
    "hgks_slab_reduce_sum", "hgks_set_stream", "hgks_get_stream", "hgks_synchronize",
    "hgks_launch_count", "hgks_set_kernel_timing", "hgks_kernel_times", "hgks_kernel_times_stage", "hgks_set_graphs", "hgks_set_grid_cap", "hgks_set_race_shake", "hgks_set_face_tma", "hgks_set_cell_tma",
    "hgks_measure_fp64_peak",
]

HGKS_REDUCE_MIN_U64, HGKS_REDUCE_SUM_F64 = 0, 1


class HgksConfig(ctypes.Structure):
    _fields_ = [
        ("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
        ("xs", _dp), ("ys", _dp), ("zs", _dp),
        ("degree", ctypes.c_int), ("dim", ctypes.c_int),
        ("gamma", ctypes.c_double), ("mu", ctypes.c_double),
        ("device", ctypes.c_int), ("z_begin", ctypes.c_int), ("z_count", ctypes.c_int),
    ]


HALO_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int)
REDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int)
RECORD_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double)

_lib = None


def load():
    """Load libhgks_b200.so (raises if absent: the product has no CPU path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -m paper_2202_13821_b200.build` "
            "(the CUDA library is required — there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    sp = ctypes.c_void_p
    L.hgks_abi_version.restype = ctypes.c_int
    L.hgks_create.argtypes = [ctypes.POINTER(HgksConfig), ctypes.POINTER(sp)]
    L.hgks_destroy.argtypes = [sp]
    L.hgks_destroy.restype = None
    L.hgks_last_error.argtypes = [sp]
    L.hgks_last_error.restype = ctypes.c_char_p
    L.hgks_error_info.argtypes = [sp, _ip, _ip, _lp, _dp]
    L.hgks_error_info.restype = None
    L.hgks_num_basis.argtypes = [sp]
    L.hgks_num_coeffs.argtypes = [sp]
    L.hgks_num_coeffs.restype = ctypes.c_long
    L.hgks_face_points.argtypes = [sp, ctypes.c_int]
    L.hgks_set_state.argtypes = [sp, _dp, ctypes.c_double]
    L.hgks_get_state.argtypes = [sp, _dp, _dp]
    L.hgks_residual.argtypes = [sp, _dp, ctypes.c_double, _dp, _dp, _dp, _dp, _dp]
    L.hgks_apply_inverse_mass.argtypes = [sp, _dp, _dp]
    L.hgks_compute_dt.argtypes = [sp, ctypes.c_double, _dp]
    L.hgks_compute_dt_k.argtypes = [sp, ctypes.c_double, ctypes.c_int, _dp]
    L.hgks_step.argtypes = [sp, ctypes.c_double]
    L.hgks_two_stage_step_host.argtypes = [sp, _dp, ctypes.c_double]
    L.hgks_two_stage_step_host_streamed.argtypes = [sp, _dp, ctypes.c_double, ctypes.c_int]
    L.hgks_advance.argtypes = [sp, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, _ip]
    L.hgks_advance_records.argtypes = [sp, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_int, RECORD_FN, sp, _ip]
    L.hgks_set_count_fluxes.argtypes = [sp, ctypes.c_int]
    L.hgks_set_count_fluxes.restype = None
    L.hgks_flux_evaluations.argtypes = [sp]
    L.hgks_flux_evaluations.restype = ctypes.c_long
    L.hgks_project_case.argtypes = [sp, ctypes.c_char_p, ctypes.c_double]
    L.hgks_tgv_diagnostics.argtypes = [sp, _dp, _dp, _dp]
    L.hgks_error_norms.argtypes = [sp, ctypes.c_char_p, ctypes.c_double, _dp]
    L.hgks_projection_npts.argtypes = [sp]
    L.hgks_project_samples.argtypes = [sp, _dp, ctypes.c_double]
    L.hgks_error_norms_samples.argtypes = [sp, _dp, _dp]
    L.hgks_halo_bytes.argtypes = [sp]
    L.hgks_halo_bytes.restype = ctypes.c_long
    L.hgks_halo_buffers.argtypes = [sp, _u64p, _u64p, _u64p, _u64p]
    L.hgks_halo_pack.argtypes = [sp, ctypes.c_int]
    L.hgks_halo_unpack.argtypes = [sp, ctypes.c_int]
    L.hgks_step_phase.argtypes = [sp, ctypes.c_double, ctypes.c_int]
    L.hgks_measure_fp64_peak.argtypes = [ctypes.c_int, ctypes.c_double, _dp]
    L.hgks_set_halo_exchange.argtypes = [sp, HALO_FN, sp]
    L.hgks_set_halo_exchange.restype = None
    L.hgks_set_halo_exchange_split.argtypes = [sp, HALO_FN, HALO_FN, sp]
    L.hgks_set_halo_exchange_split.restype = None
    L.hgks_set_host_reduce.argtypes = [sp, REDUCE_FN, sp]
    L.hgks_set_host_reduce.restype = None
    L.hgks_nccl_unique_id.argtypes = [ctypes.c_char_p, ctypes.c_int]
    L.hgks_attach_nccl.argtypes = [sp, ctypes.c_char_p, ctypes.c_int, ctypes.c_int]
    L.hgks_attach_nccl_comm.argtypes = [sp, sp, ctypes.c_int, ctypes.c_int]
    L.hgks_slab_reduce_sum.argtypes = [sp, _dp, ctypes.c_int]
    L.hgks_set_graphs.argtypes = [sp, ctypes.c_int]
    L.hgks_set_graphs.restype = None
    L.hgks_set_grid_cap.argtypes = [sp, ctypes.c_int]
    L.hgks_set_grid_cap.restype = None
    L.hgks_set_race_shake.argtypes = [sp, ctypes.c_uint]
    L.hgks_set_race_shake.restype = None
    L.hgks_set_face_tma.argtypes = [sp, ctypes.c_int]
    L.hgks_set_face_tma.restype = None
    L.hgks_set_cell_tma.argtypes = [sp, ctypes.c_int]
    L.hgks_set_cell_tma.restype = None
    L.hgks_set_stream.argtypes = [sp, sp]
    L.hgks_get_stream.argtypes = [sp]
    L.hgks_get_stream.restype = sp
    L.hgks_synchronize.argtypes = [sp]
    L.hgks_launch_count.argtypes = [sp]
    L.hgks_launch_count.restype = ctypes.c_long
    L.hgks_set_kernel_timing.argtypes = [sp, ctypes.c_int]
    L.hgks_set_kernel_timing.restype = None
    L.hgks_kernel_times.argtypes = [sp, _dp, _dp, _dp]
    L.hgks_kernel_times_stage.argtypes = [sp, ctypes.c_int, _dp, _dp]
    _lib = L
    return L
