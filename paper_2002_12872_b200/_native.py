"""ctypes binding of the C ABI in include/dpt_b200.h (libdpt_b200.so, built in-tree).

The CUDA library is REQUIRED: there is no CPU fallback.  Importing works on a
CPU-only host (the library loads without a GPU), but creating a context there
raises NoDeviceError.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, Structure, c_char, c_double, c_int, c_int32, c_int64, c_size_t,
                    c_void_p)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DPT_LIB_PATH") or os.path.join(_HERE, "libdpt_b200.so")  # override: A/B builds
PROBLEMS_PATH = os.path.join(_HERE, "libdpt_problems.so")

DPT_MEM_HOST, DPT_MEM_DEVICE = 0, 1
DPT_DELTA_DENSE, DPT_DELTA_CSR = 0, 1

(DPT_OK, DPT_ERR_SHAPE, DPT_ERR_DEGENERATE, DPT_ERR_INVALID_ARG, DPT_ERR_CUDA, DPT_ERR_NCCL,
 DPT_ERR_NON_REAL, DPT_ERR_NO_DEVICE, DPT_ERR_TRACE, DPT_ERR_UNSUPPORTED, DPT_ERR_IO) = range(11)


class dpt_options(Structure):
    _fields_ = [("tol", c_double), ("residual_tol", c_double), ("max_iter", c_int),
                ("divergence_threshold", c_double), ("cycle_window", c_int),
                ("degeneracy_tol", c_double)]


class dpt_problem(Structure):
    _fields_ = [("n", c_int64), ("d", c_void_p), ("delta_kind", c_int), ("delta", c_void_p),
                ("rowptr", c_void_p), ("cols", c_void_p), ("vals", c_void_p), ("nnz", c_int64),
                ("lambda_", c_double), ("mem", c_int), ("is_complex", c_int), ("lambda_im", c_double)]


class dpt_report(Structure):
    _fields_ = [("status", c_int), ("iterations", c_int), ("step_norm", c_double),
                ("eigenvalue", c_double), ("residual", c_double), ("row", c_int64),
                ("device_ms", c_double), ("launches", c_int), ("eigenvalue_im", c_double)]


class dpt_error_info(Structure):
    _fields_ = [("code", c_int), ("i", c_int64), ("j", c_int64), ("ei", c_double), ("ej", c_double),
                ("message", c_char * 256), ("ei_im", c_double), ("ej_im", c_double)]


TRACE_FN = ctypes.CFUNCTYPE(c_int, c_int, c_double, c_double, c_void_p)

_lib = None
_plib = None


class dpt_mm_matrix(Structure):
    _fields_ = [("rows", c_int64), ("cols", c_int64), ("is_sparse", c_int), ("is_complex", c_int),
                ("nnz", c_int64), ("rowptr", c_void_p), ("colidx", c_void_p), ("vals", c_void_p),
                ("store", c_void_p)]


class dpt_scan_grid(Structure):
    _fields_ = [("re_min", c_double), ("re_max", c_double), ("im_min", c_double), ("im_max", c_double),
                ("res_re", c_int64), ("res_im", c_int64)]


DPT_SCAN_FULL, DPT_SCAN_SINGLE_ROW = 0, 1


def lib() -> ctypes.CDLL:
    """Load libdpt_b200.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C "
                              "paper_2002_12872_b200/csrc); the DPT path has no CPU fallback")
        L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        P, D, I, I64 = POINTER, c_double, c_int, c_int64
        L.dpt_ctx_create.argtypes = [c_int, P(c_void_p), P(dpt_error_info)]
        L.dpt_ctx_destroy.argtypes = [c_void_p]
        L.dpt_ctx_set_comm.argtypes = [c_void_p, c_int, c_int, c_void_p, c_size_t, P(dpt_error_info)]
        L.dpt_nccl_unique_id.argtypes = [c_void_p, c_size_t, P(dpt_error_info)]
        L.dpt_ctx_stream.argtypes = [c_void_p]
        L.dpt_ctx_stream.restype = c_void_p
        L.dpt_ctx_launch_count.argtypes = [c_void_p]
        L.dpt_ctx_launch_count.restype = c_int64
        L.dpt_ctx_graph_stats.argtypes = [c_void_p, P(c_int64), P(c_int64)]
        L.dpt_ctx_graph_stats.restype = None
        L.dpt_ctx_set_loopback.argtypes = [P(c_void_p), c_int, P(dpt_error_info)]
        L.dpt_ctx_set_loopback.restype = c_int
        L.dpt_options_default.argtypes = [P(dpt_options)]
        L.dpt_status_string.argtypes = [c_int]
        L.dpt_status_string.restype = ctypes.c_char_p
        L.dpt_iterate_full.argtypes = [c_void_p, P(dpt_problem), P(dpt_options), TRACE_FN, c_void_p,
                                       c_void_p, c_void_p, c_void_p, c_int, P(dpt_report),
                                       P(dpt_error_info)]
        L.dpt_iterate_ramped.argtypes = [c_void_p, P(dpt_problem), D, P(dpt_options), TRACE_FN,
                                         c_void_p, c_void_p, c_void_p, c_void_p, c_int, P(dpt_report),
                                         P(dpt_error_info)]
        L.dpt_iterate_fixed.argtypes = [c_void_p, P(dpt_problem), I, D, c_void_p, c_int,
                                        P(dpt_report), P(dpt_error_info)]
        L.dpt_step_full.argtypes = [c_void_p, P(dpt_problem), c_void_p, D, c_void_p, c_int,
                                    P(dpt_error_info)]
        L.dpt_iterate_single.argtypes = [c_void_p, P(dpt_problem), I64, P(dpt_options), D, TRACE_FN,
                                         c_void_p, c_void_p, c_int, P(dpt_report), P(dpt_error_info)]
        L.dpt_dominant_eigenpair.argtypes = [c_void_p, P(dpt_problem), P(dpt_options), c_void_p,
                                             c_void_p, c_int, P(dpt_report), P(dpt_error_info)]
        L.dpt_step_single.argtypes = [c_void_p, P(dpt_problem), c_void_p, I64, D, c_void_p, c_int,
                                      P(dpt_error_info)]
        L.dpt_eigenvalue_of.argtypes = [c_void_p, P(dpt_problem), c_void_p, I64, D, P(c_double),
                                        c_int, P(dpt_error_info)]
        L.dpt_iterate_fixed_c.argtypes = [c_void_p, P(dpt_problem), I, D, D, c_void_p, c_int, P(dpt_report),
                                          P(dpt_error_info)]
        L.dpt_step_full_gap_c.argtypes = [c_void_p, P(dpt_problem), c_void_p, c_void_p, D, D, c_void_p, c_int,
                                          P(dpt_error_info)]
        L.dpt_step_single_gap_c.argtypes = [c_void_p, P(dpt_problem), c_void_p, I64, c_void_p, D, D, c_void_p,
                                            c_int, P(dpt_error_info)]
        L.dpt_eigenvalue_of_c.argtypes = [c_void_p, P(dpt_problem), c_void_p, I64, D, D, c_void_p, c_int,
                                          P(dpt_error_info)]
        L.dpt_step_full_gap.argtypes = [c_void_p, P(dpt_problem), c_void_p, c_void_p, D, c_void_p, c_int,
                                        P(dpt_error_info)]
        L.dpt_step_single_gap.argtypes = [c_void_p, P(dpt_problem), c_void_p, I64, c_void_p, D, c_void_p, c_int,
                                          P(dpt_error_info)]
        L.dpt_readoffs.argtypes = [c_void_p, P(dpt_problem), c_void_p, c_void_p, c_void_p, c_int,
                                   P(dpt_error_info)]
        L.dpt_plan_create.argtypes = [c_void_p, P(dpt_problem), c_int, I64, D, P(c_void_p), P(dpt_error_info)]
        L.dpt_plan_destroy.argtypes = [c_void_p]
        L.dpt_plan_begin.argtypes = [c_void_p, P(dpt_error_info)]
        L.dpt_plan_steps.argtypes = [c_void_p, c_int, P(c_double), P(dpt_error_info)]
        L.dpt_plan_read.argtypes = [c_void_p, c_void_p, c_int, P(dpt_error_info)]
        L.dpt_plan_stats.argtypes = [c_void_p, c_void_p, P(dpt_error_info)]
        L.dpt_probe_fp64_peak.argtypes = [c_int, P(c_double), P(dpt_error_info)]
        L.dpt_check_degenerate.argtypes = [I64, c_void_p, D, P(c_int64), P(c_int64)]
        L.dpt_spectral_spread.argtypes = [I64, c_void_p]
        L.dpt_spectral_spread.restype = D
        L.dpt_effective_window.argtypes = [c_int, I64]
        L.dpt_matmul_dense.argtypes = [c_void_p, c_int64, c_int64, c_int64, c_int, c_void_p, c_void_p, c_void_p,
                                       c_int, P(dpt_error_info)]
        L.dpt_solve_linear_multi.argtypes = [c_void_p, c_int64, c_int64, c_int, c_void_p, c_void_p, c_void_p, c_int,
                                             P(dpt_error_info)]
        L.dpt_homotopy_solve.argtypes = [c_void_p, P(dpt_problem), c_int, P(dpt_options), c_void_p, c_void_p,
                                         c_void_p, c_int, P(dpt_report), P(dpt_error_info)]
        L.dpt_mm_read.argtypes = [ctypes.c_char_p, c_int, P(dpt_mm_matrix), P(dpt_error_info)]
        L.dpt_mm_free.argtypes = [P(dpt_mm_matrix)]
        L.dpt_mm_write_dense.argtypes = [ctypes.c_char_p, I64, I64, c_void_p, c_int, c_int, P(dpt_error_info)]
        L.dpt_mm_write_csr.argtypes = [ctypes.c_char_p, I64, I64, c_void_p, c_void_p, c_void_p, c_int, c_int,
                                       P(dpt_error_info)]
        L.dpt_scan_domain.argtypes = [c_void_p, P(dpt_problem), P(dpt_scan_grid), c_int, I64, D, P(dpt_options),
                                      c_void_p, c_void_p, P(dpt_error_info)]
        L.dpt_sm_state_bytes.restype = c_size_t
        L.dpt_sm_init.argtypes = [c_void_p, c_void_p, P(dpt_options), c_int, c_int]
        L.dpt_sm_decide_host.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_void_p]
        L.dpt_sm_query.argtypes = [c_void_p, P(c_int), P(c_int), P(c_int), P(c_int), P(c_int),
                                   P(c_int), P(c_double)]
        _lib = L
    return _lib


def problems_lib() -> ctypes.CDLL:
    global _plib
    if _plib is None:
        if not os.path.exists(PROBLEMS_PATH):
            raise ImportError(f"{PROBLEMS_PATH} is missing: run __graft_entry__.build()")
        L = ctypes.CDLL(PROBLEMS_PATH)
        L.dpt_gen_rng_u64.argtypes = [ctypes.c_uint64, ctypes.c_char_p, c_int64]
        L.dpt_gen_rng_u64.restype = ctypes.c_uint64
        L.dpt_gen_theta_linear.argtypes = [c_int64, c_double, c_void_p]
        L.dpt_gen_theta_uniform_sorted.argtypes = [c_int64, ctypes.c_uint64, c_double, c_double,
                                                   c_void_p]
        L.dpt_gen_dense_normal.argtypes = [c_int64, ctypes.c_uint64, ctypes.c_char_p, c_int, c_void_p]
        L.dpt_gen_csr_sym_bernoulli.argtypes = [c_int64, ctypes.c_uint64, c_double, c_void_p,
                                                c_void_p, c_void_p]
        L.dpt_gen_csr_sym_bernoulli.restype = c_int64
        L.dpt_gen_csr_fixed_per_row.argtypes = [c_int64, ctypes.c_uint64, c_int, c_void_p, c_void_p,
                                                c_void_p]
        L.dpt_gen_csr_fixed_per_row.restype = c_int64
        L.dpt_gen_random_uniform.argtypes = [c_int64, ctypes.c_uint64, c_void_p, c_void_p]
        L.dpt_gen_oscillator.argtypes = [c_int64, c_void_p, c_void_p]
        _plib = L
    return _plib
