"""ctypes binding of librcg_b200.so (the C-ABI declared in include/rcg_b200.h).

The library is built in-tree by ``make -C paper_2203_08498_b200/csrc`` (``__graft_entry__.build``).
There is no fallback: if the shared object is missing this module raises at import, and every
compute call returns RCG_E_CUDA when no sm_100 GPU is present.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RCG_LIB_PATH") or os.path.join(_HERE, "librcg_b200.so")  # override: dev A/B only

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make -C {_HERE}/csrc` "
        "(the CUDA path has no CPU fallback)"
    )

lib = C.CDLL(LIB_PATH)

RCG_OK, RCG_E_INVALID, RCG_E_BREAKDOWN, RCG_E_PARSE, RCG_E_CUDA = 0, 1, 2, 3, 4
RCG_PREC_IDENTITY, RCG_PREC_IC, RCG_PREC_SC = 0, 1, 2
RCG_PAYLOAD_X, RCG_PAYLOAD_R = 0, 1
RCG_SAMPLER_A, RCG_SAMPLER_B = 0, 1
RCG_BASIS_DEFLATION, RCG_BASIS_SC = 0, 1
RCG_GEN_POISSON7, RCG_GEN_FV7_CONTRAST, RCG_GEN_Q1_27PT, RCG_GEN_KNN = 0, 1, 2, 3
RCG_METHOD_CG, RCG_METHOD_ICCG, RCG_METHOD_ES_SC_ICCG, RCG_METHOD_ES_D_ICCG = 0, 1, 2, 3

vp = C.c_void_p
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)

# host transport callbacks (rcg_comm_create_host)
HostAllreduceFn = C.CFUNCTYPE(C.c_int, vp, dp, C.c_int)
HostExchangeFn = C.CFUNCTYPE(C.c_int, vp, dp, i64p, i64p, dp, i64p, i64p, C.c_int)


class SolverConfig(C.Structure):
    _fields_ = [("eps", C.c_double), ("max_iter", C.c_int), ("record_history", C.c_int)]


class SolveReport(C.Structure):
    _fields_ = [
        ("iterations", C.c_int),
        ("converged", C.c_int),
        ("wall_time", C.c_double),
        ("cap", C.c_int),
        ("history", dp),
        ("alphas", dp),
        ("betas", dp),
    ]


class Prec(C.Structure):
    _fields_ = [("kind", C.c_int), ("ic", vp), ("sc", vp)]


class CondEstimate(C.Structure):
    _fields_ = [
        ("lambda_max", C.c_double),
        ("lambda_min", C.c_double),
        ("kappa", C.c_double),
        ("power_iterations", C.c_int),
        ("power_unsettled", C.c_int),
        ("lambda_min_available", C.c_int),
        ("nritz", C.c_int),
        ("ritz_values", dp),
        ("lanczos_lambda_min", C.c_double),
        ("lanczos_lambda_max", C.c_double),
        ("lanczos_kappa", C.c_double),
    ]


class GenParams(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("grid", C.c_int32),
        ("inclusions", C.c_int),
        ("inclusion_size", C.c_int),
        ("contrast", C.c_double),
        ("sigma", C.c_double),
        ("knn_k", C.c_int),
        ("seed", C.c_uint64),
    ]


class SlabPlanC(C.Structure):
    _fields_ = [
        ("row_begin", C.c_int32), ("row_end", C.c_int32), ("nloc", C.c_int32), ("nhalo", C.c_int32),
        ("nnz", C.c_int64), ("row_start", i32p), ("col_idx", i32p), ("values", dp), ("halo_global", i32p),
        ("recv_count", i32p), ("send_count", i32p), ("send_idx", i32p), ("nparts", C.c_int), ("part", C.c_int),
    ]


class SeqConfig(C.Structure):
    _fields_ = [("eps", C.c_double), ("max_iter", C.c_int), ("sampling", C.c_int), ("m", C.c_int),
                ("theta", C.c_double), ("keep_count", C.c_int), ("batch", C.c_int), ("memory", C.c_int)]


class SeqReport(C.Structure):
    _fields_ = [("iterations", ip), ("converged", ip), ("wall_time", dp), ("true_relres", dp),
                ("ritz_values", dp), ("ritz_cap", C.c_int), ("m_bar", C.c_int), ("m_tilde", C.c_int),
                ("theta_used", C.c_double), ("w_build_time", C.c_double), ("avg_iterations", C.c_double),
                ("avg_wall_time", C.c_double), ("setup_time", C.c_double), ("acceleration_inactive", C.c_int),
                ("lambda_min", dp), ("lambda_max", dp), ("kappa", dp)]


def _sig(name, restype, *args):
    f = getattr(lib, name)
    f.restype = restype
    f.argtypes = list(args)
    return f


# every symbol declared in include/rcg_b200.h, with its ctypes signature
SIGNATURES = {
    "rcg_last_error": (C.c_char_p,),
    "rcg_build_info": (C.c_char_p,),
    "rcg_ctx_create": (C.c_int, C.c_int, C.POINTER(vp)),
    "rcg_ctx_destroy": (None, vp),
    "rcg_ctx_synchronize": (C.c_int, vp),
    "rcg_ctx_launch_count": (C.c_int64, vp),
    "rcg_ctx_set_profiling": (C.c_int, vp, C.c_int),
    "rcg_ctx_set_profiling_mask": (C.c_int, vp, C.c_uint),
    "rcg_ctx_set_sweep_kernel": (C.c_int, vp, C.c_int),
    "rcg_ctx_event_record": (C.c_int, vp, C.c_int),
    "rcg_ctx_event_elapsed": (C.c_int, vp, C.c_int, C.c_int, dp),
    "rcg_ctx_kernel_stats": (C.c_int, vp, C.c_int, dp, i64p),
    "rcg_ctx_kernel_units": (C.c_int, vp, C.c_int, i64p),
    "rcg_ctx_reset_stats": (None, vp),
    "rcg_matrix_create": (C.c_int, vp, C.c_int32, vp, vp, vp, C.c_int, C.POINTER(vp)),
    "rcg_matrix_destroy": (None, vp),
    "rcg_matrix_n": (C.c_int32, vp),
    "rcg_matrix_nnz": (C.c_int64, vp),
    "rcg_matrix_values": (C.c_int, vp, vp, vp),
    "rcg_spmv": (C.c_int, vp, vp, vp, vp),
    "rcg_spmv_dual": (C.c_int, vp, vp, vp, vp, vp, vp),
    "rcg_diagonal_scale": (C.c_int, vp, vp, C.POINTER(vp), vp),
    "rcg_ic0_factorize": (C.c_int, vp, C.c_int32, vp, vp, vp, C.c_double, C.c_int, C.POINTER(vp)),
    "rcg_ic0_factorize_device": (C.c_int, vp, vp, C.c_double, C.c_int, C.POINTER(vp)),
    "rcg_ic_create": (C.c_int, vp, C.c_int32, C.c_int, vp, vp, vp, vp, vp, vp, vp, vp, C.c_double, C.POINTER(vp)),
    "rcg_ic_destroy": (None, vp),
    "rcg_ic_info": (C.c_int, vp, i64p, dp, i32p, i32p),
    "rcg_ic_export": (C.c_int, vp, vp, vp, vp, vp, vp, vp, vp, vp),
    "rcg_ic_apply": (C.c_int, vp, vp, vp, vp),
    "rcg_tall_create": (C.c_int, vp, C.c_int32, C.c_int, vp, C.POINTER(vp)),
    "rcg_tall_create_cols": (C.c_int, vp, C.c_int32, C.c_int, C.POINTER(vp), C.POINTER(vp)),
    "rcg_tall_destroy": (None, vp),
    "rcg_tall_k": (C.c_int, vp),
    "rcg_tall_n": (C.c_int32, vp),
    "rcg_tall_download": (C.c_int, vp, vp, vp),
    "rcg_mgs_orthonormalize": (C.c_int, vp, vp, C.c_double, C.POINTER(vp)),
    "rcg_sampler_create": (C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int32, C.POINTER(vp)),
    "rcg_sampler_destroy": (None, vp),
    "rcg_sampler_offer": (C.c_int, vp, vp, C.c_int, C.c_double, vp),
    "rcg_sampler_state": (C.c_int, vp, vp, vp),
    "rcg_sampler_slot": (C.c_int, vp, vp, C.c_int, vp),
    "rcg_harvest_errors": (C.c_int, vp, vp, vp, C.POINTER(vp)),
    "rcg_harvest_columns": (C.c_int, vp, vp, C.c_int32, C.c_int, C.POINTER(vp), C.POINTER(vp)),
    "rcg_harvest_stored": (C.c_int, vp, vp, C.POINTER(vp)),
    "rcg_rayleigh_ritz": (C.c_int, vp, vp, vp, vp, C.POINTER(vp)),
    "rcg_build_aux_matrix": (C.c_int, vp, vp, vp, C.c_double, C.c_int, ip, vp, dp, C.POINTER(vp)),
    "rcg_basis_create": (C.c_int, vp, vp, vp, C.c_int, C.POINTER(vp)),
    "rcg_basis_destroy": (None, vp),
    "rcg_basis_k": (C.c_int, vp),
    "rcg_basis_create_from": (C.c_int, vp, C.c_int32, C.c_int, C.POINTER(vp), C.POINTER(vp), vp, C.c_int, C.POINTER(vp)),
    "rcg_basis_export": (C.c_int, vp, vp, vp, vp),
    "rcg_project_pt": (C.c_int, vp, vp, vp, vp),
    "rcg_project_p": (C.c_int, vp, vp, vp, vp),
    "rcg_direct_component": (C.c_int, vp, vp, vp, vp),
    "rcg_prec_apply": (C.c_int, vp, C.POINTER(Prec), vp, vp),
    "rcg_pcg_solve": (C.c_int, vp, vp, vp, C.POINTER(Prec), vp, C.POINTER(SolverConfig), vp, C.c_int,
                      C.POINTER(SolveReport)),
    "rcg_deflated_pcg_solve": (C.c_int, vp, vp, vp, C.POINTER(Prec), vp, vp, C.POINTER(SolverConfig),
                               C.POINTER(SolveReport)),
    "rcg_pcg_solve_batch": (C.c_int, vp, vp, vp, C.POINTER(Prec), vp, C.POINTER(SolverConfig), C.c_int,
                            C.POINTER(SolveReport)),
    "rcg_deflated_pcg_solve_batch": (C.c_int, vp, vp, vp, C.POINTER(Prec), vp, vp, C.POINTER(SolverConfig), C.c_int,
                                     C.POINTER(SolveReport)),
    "rcg_pcg_with_condest": (C.c_int, vp, vp, vp, C.POINTER(Prec), vp, C.POINTER(SolverConfig), C.c_int,
                             C.c_uint64, C.POINTER(SolveReport), C.POINTER(CondEstimate)),
    "rcg_lanczos_extremes": (C.c_int, C.c_int, vp, vp, dp, dp),
    "rcg_generate": (C.c_int, C.POINTER(GenParams), i32p, i64p, C.POINTER(i32p), C.POINTER(i32p), C.POINTER(dp)),
    "rcg_matrix_generate": (C.c_int, vp, C.POINTER(GenParams), C.POINTER(vp)),
    "rcg_matrix_export": (C.c_int, vp, vp, vp, vp, vp),
    "rcg_uniform_pm1": (None, C.c_uint64, C.c_uint64, C.c_int64, vp),
    "rcg_normal": (None, C.c_uint64, C.c_uint64, C.c_int64, vp),
    "rcg_host_free": (None, vp),
    "rcg_level_depth": (C.c_int, C.c_int32, vp, vp, i32p),
    "rcg_multicolor_order": (C.c_int, C.c_int32, vp, vp, vp, i32p),
    "rcg_permute_symmetric": (C.c_int, C.c_int32, vp, vp, vp, vp, C.POINTER(i32p), C.POINTER(i32p),
                              C.POINTER(dp)),
    "rcg_slab_plan_create": (C.c_int, C.c_int32, vp, vp, vp, C.c_int, C.c_int, C.POINTER(SlabPlanC)),
    "rcg_slab_plan_free": (None, C.POINTER(SlabPlanC)),
    "rcg_dslab_create": (C.c_int, vp, C.POINTER(SlabPlanC), vp, C.POINTER(vp)),
    "rcg_dslab_destroy": (None, vp),
    "rcg_comm_nccl_unique_id": (C.c_int, vp),
    "rcg_comm_create_nccl": (C.c_int, vp, C.c_int, C.c_int, C.POINTER(vp)),
    "rcg_comm_create_loopback": (C.c_int, C.c_int, C.POINTER(vp)),
    "rcg_comm_create_host": (C.c_int, C.c_int, C.c_int, HostAllreduceFn, HostExchangeFn, vp, C.POINTER(vp)),
    "rcg_comm_destroy": (None, vp),
    "rcg_dist_pcg_solve": (C.c_int, vp, C.c_int, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                           C.POINTER(SolverConfig), C.POINTER(SolveReport)),
    "rcg_seq_prepare": (C.c_int, vp, vp, C.c_int, C.c_int, C.POINTER(vp)),
    "rcg_seq_destroy": (None, vp),
    "rcg_seq_run": (C.c_int, vp, C.c_int, vp, vp, C.POINTER(SeqConfig), C.POINTER(SeqReport)),
    "rcg_dbasis_create": (C.c_int, vp, C.c_int, C.POINTER(vp), C.POINTER(vp), C.c_int, C.c_int, C.POINTER(vp)),
    "rcg_dbasis_destroy": (None, vp),
    "rcg_dist_solve_batch": (C.c_int, vp, vp, vp, vp, vp, C.POINTER(SolverConfig), C.c_int, C.POINTER(SolveReport)),
    "rcg_dist_solve": (C.c_int, vp, C.c_int, C.POINTER(vp), vp, C.POINTER(vp), C.POINTER(vp),
                       C.POINTER(SolverConfig), C.POINTER(SolveReport)),
    "rcg_dist_pcg_solve_sampled": (C.c_int, vp, C.c_int, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                   C.POINTER(SolverConfig), C.POINTER(SolveReport)),
    "rcg_dist_recycle": (C.c_int, vp, C.c_int, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.c_double, C.c_int, C.c_int,
                         ip, vp, dp, ip, C.POINTER(vp)),
}

for _name, (_res, *_args) in SIGNATURES.items():
    _sig(_name, _res, *_args)


class RcgError(RuntimeError):
    """Base of the mapped status codes."""


class InvalidArgument(RcgError, ValueError):
    """std::invalid_argument"""


class BreakdownError(RcgError):
    """recycg::BreakdownError"""


class ParseError(RcgError):
    """recycg::ParseError"""


class CudaError(RcgError):
    """CUDA / device failure (no CPU fallback exists)"""


_ERRS = {RCG_E_INVALID: InvalidArgument, RCG_E_BREAKDOWN: BreakdownError, RCG_E_PARSE: ParseError,
         RCG_E_CUDA: CudaError}


def check(status: int) -> None:
    if status != RCG_OK:
        msg = lib.rcg_last_error().decode(errors="replace")
        raise _ERRS.get(status, RcgError)(msg)
