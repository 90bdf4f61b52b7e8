"""Python mirror of the reference's DPT solver API (proj/include/dynspec/dpt.hpp).

Same names, argument meaning and error behaviour as the reference's C++ free
functions, over the C ABI of libdpt_b200.so (include/dpt_b200.h):

  iterate_full(p, opts, trace)          dpt.hpp:74-83
  iterate_ramped(p, alpha, opts, trace) dpt.hpp:85-92
  iterate_fixed(p, k, lam)              dpt.hpp:94-96
  step_full(a, p, lam)                  dpt.hpp:51-57 (theta from p.d, Delta from p)
  iterate_single(p, row, opts, ramp_alpha, trace)   dpt.hpp:107-111
  dominant_eigenpair(p, opts)           dpt.hpp:113-129
  step_single(z, row, p, lam)           dpt.hpp:59-66
  eigenvalue_of(z, row, p, lam)         dpt.hpp:68-72

Non-convergence is a status (ConvergenceStatus), never an exception; the
exceptions mirror the reference's: ShapeError, DegenerateSpectrum(i, j, ei, ej),
ValueError for std::invalid_argument.  Arrays are real FP64, row-major.

Every call runs on the GPU; without a CUDA device it raises NoDeviceError (the
path has no CPU fallback).
"""
from __future__ import annotations

import ctypes
import enum
import threading
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _native as N


class ConvergenceStatus(enum.IntEnum):  # dpt.hpp:13-18
    Converged = 0
    BoundedNonConverged = 1
    Diverged = 2
    MaxIterations = 3


def to_string(s: ConvergenceStatus) -> str:  # dpt.cpp:297-309
    return N.lib().dpt_status_string(int(s)).decode()


class ShapeError(ValueError):
    """ShapeError (matrix.hpp:16-19)."""


class DegenerateSpectrum(RuntimeError):
    """DegenerateSpectrum (partition.hpp:13-26): carries the offending pair."""

    def __init__(self, msg, i, j, ei, ej):
        super().__init__(msg)
        self.i, self.j, self.ei, self.ej = int(i), int(j), ei, ej

    def first(self):
        return self.i

    def second(self):
        return self.j


class IoError(RuntimeError):
    """IoError (matrix_market.hpp:10-13)."""


class NoDeviceError(RuntimeError):
    """No CUDA device: the DPT path has no CPU fallback."""


class DeviceError(RuntimeError):
    pass


class TraceAborted(RuntimeError):
    pass


@dataclass
class IterationOptions:  # dpt.hpp:22-31
    tol: float = 1e-12
    residual_tol: float = 1e-10
    max_iter: int = 10000
    divergence_threshold: float = 1e8
    cycle_window: int = 16
    degeneracy_tol: float = 1e-12

    def _c(self) -> N.dpt_options:
        return N.dpt_options(self.tol, self.residual_tol, int(self.max_iter),
                             self.divergence_threshold, int(self.cycle_window), self.degeneracy_tol)


@dataclass
class CsrMatrix:
    """CSR with int64 row offsets, int32 sorted columns, FP64 values (matrix.hpp:73-106).
    `n` rows; `ncols` columns when not square (Matrix Market files)."""
    n: int
    rowptr: np.ndarray
    cols: np.ndarray
    vals: np.ndarray
    ncols: Optional[int] = None

    @property
    def nnz(self) -> int:
        return int(self.vals.shape[0])

    def todense(self) -> np.ndarray:
        out = np.zeros((self.n, self.ncols or self.n), dtype=np.asarray(self.vals).dtype)
        for i in range(self.n):
            s, e = int(self.rowptr[i]), int(self.rowptr[i + 1])
            out[i, self.cols[s:e]] = self.vals[s:e]
        return out


@dataclass
class PartitionedProblem:  # partition.hpp:43-50 (delta_t is not needed on the device)
    d: object            # [n] levels (numpy or torch CUDA tensor)
    delta: object        # dense [n, n] (numpy / torch CUDA) or CsrMatrix (numpy / torch CUDA parts)
    lam: float = 1.0

    def size(self) -> int:
        return int(self.d.shape[0])


@dataclass
class EigenIterate:  # dpt.hpp:34-37
    a: object
    k: int = 0


@dataclass
class ConvergenceReport:  # dpt.hpp:39-46
    state: EigenIterate
    eigenvalues: object
    status: ConvergenceStatus
    iterations: int
    residuals: object
    step_norm: float
    device_ms: float = 0.0


@dataclass
class SingleRowReport:  # dpt.hpp:98-105
    z: object
    eigenvalue: float
    status: ConvergenceStatus
    iterations: int
    residual: float
    step_norm: float
    device_ms: float = 0.0


@dataclass
class DominantEigenpair:  # dpt.hpp:113-122
    row: int
    z_chart: object
    z_unit: object
    eigenvalue: float
    status: ConvergenceStatus
    iterations: int
    residual: float
    step_norm: float
    device_ms: float = 0.0


# ---------------------------------------------------------------- context ----
class Context:
    """One CUDA stream + (optionally) one NCCL communicator (dpt_ctx)."""

    def __init__(self, device: int = 0):
        err = N.dpt_error_info()
        h = ctypes.c_void_p()
        rc = N.lib().dpt_ctx_create(device, ctypes.byref(h), ctypes.byref(err))
        if rc == N.DPT_ERR_NO_DEVICE:
            raise NoDeviceError(err.message.decode())
        _raise(rc, err)
        self.handle = h
        self.device = device

    def set_comm(self, rank: int, world: int, nccl_id: bytes):
        err = N.dpt_error_info()
        buf = ctypes.create_string_buffer(nccl_id, len(nccl_id))
        _raise(N.lib().dpt_ctx_set_comm(self.handle, rank, world, buf, len(nccl_id), ctypes.byref(err)), err)

    @staticmethod
    def set_loopback(ctxs) -> None:
        """TEST-ONLY: make these contexts (one device) ranks 0..len-1 of a
        sharded group whose collectives are in-process (dpt_ctx_set_loopback);
        drive each rank from its own thread with the same calls."""
        arr = (ctypes.c_void_p * len(ctxs))(*[c.handle for c in ctxs])
        err = N.dpt_error_info()
        _raise(N.lib().dpt_ctx_set_loopback(arr, len(ctxs), ctypes.byref(err)), err)

    @staticmethod
    def nccl_unique_id() -> bytes:
        err = N.dpt_error_info()
        buf = ctypes.create_string_buffer(128)
        _raise(N.lib().dpt_nccl_unique_id(buf, 128, ctypes.byref(err)), err)
        return buf.raw

    @property
    def stream_ptr(self) -> int:
        return N.lib().dpt_ctx_stream(self.handle) or 0

    @property
    def launches(self) -> int:
        return int(N.lib().dpt_ctx_launch_count(self.handle))

    @property
    def graph_stats(self):
        """(hits, misses) of this context's device-loop graph cache."""
        h, m = ctypes.c_int64(0), ctypes.c_int64(0)
        N.lib().dpt_ctx_graph_stats(self.handle, ctypes.byref(h), ctypes.byref(m))
        return int(h.value), int(m.value)

    def close(self):
        if self.handle:
            N.lib().dpt_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()


def default_context(device: int = 0) -> Context:
    """Per-thread context (the reference's functions are reentrant)."""
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


def _raise(rc: int, err: N.dpt_error_info):
    if rc == N.DPT_OK:
        return
    msg = err.message.decode(errors="replace")
    if rc == N.DPT_ERR_SHAPE:
        raise ShapeError(msg)
    if rc == N.DPT_ERR_DEGENERATE:
        ei = complex(err.ei, err.ei_im) if err.ei_im else err.ei
        ej = complex(err.ej, err.ej_im) if err.ej_im else err.ej
        raise DegenerateSpectrum(msg, err.i, err.j, ei, ej)
    if rc in (N.DPT_ERR_INVALID_ARG, N.DPT_ERR_NON_REAL):
        raise ValueError(msg)
    if rc == N.DPT_ERR_NO_DEVICE:
        raise NoDeviceError(msg)
    if rc == N.DPT_ERR_TRACE:
        raise TraceAborted(msg)
    if rc == N.DPT_ERR_IO:
        raise IoError(msg)
    raise DeviceError(f"dpt error {rc}: {msg}")


# ------------------------------------------------------------ marshalling ----
def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _ptr(x) -> int:
    if _is_torch(x):
        return x.data_ptr()
    return x.ctypes.data


def _host(x, dtype):
    a = np.ascontiguousarray(np.asarray(x, dtype=dtype))
    return a


def _is_complex_dtype(x) -> bool:
    if _is_torch(x):
        return x.is_complex()
    return np.iscomplexobj(x)


def _has_imag(x) -> bool:
    if _is_torch(x):
        return bool(x.is_complex() and (x.imag != 0).any().item())
    return bool(np.iscomplexobj(x) and np.any(np.imag(x) != 0))


class _Marshal:
    """Keeps the arrays of one call alive and builds the dpt_problem.

    Real inputs (or complex dtypes whose imaginary parts are all zero) run the
    real FP64 kernels -- the reference's imaginary parts would stay exactly 0;
    inputs with a nonzero imaginary part run the complex FP64 path
    (std::complex<double> interleaved layout).  `cdtype` records whether the
    caller passed complex data, so outputs come back complex like the
    reference's std::complex results."""

    def __init__(self, p: PartitionedProblem, extra_complex=False):
        self.keep = []
        d, delta, lam = p.d, p.delta, p.lam
        vals = delta.vals if isinstance(delta, CsrMatrix) else delta
        self.cdtype = (_is_complex_dtype(d) or _is_complex_dtype(vals) or np.iscomplexobj(np.asarray(lam))
                       or extra_complex)
        self.cplx = bool(_has_imag(d) or _has_imag(vals) or (np.iscomplexobj(np.asarray(lam)) and np.imag(lam) != 0)
                         or extra_complex)
        self.device = _is_torch(d) and d.is_cuda
        n = int(d.shape[0])
        if len(d.shape) != 1:
            raise ShapeError("make_problem: diagonal must be a vector")
        self.n = n
        prob = N.dpt_problem()
        prob.n = n
        prob.d = self._arr(d)
        prob.lambda_ = float(np.real(lam))
        prob.lambda_im = float(np.imag(lam)) if self.cplx else 0.0
        prob.is_complex = 1 if self.cplx else 0
        prob.mem = N.DPT_MEM_DEVICE if self.device else N.DPT_MEM_HOST
        if isinstance(delta, CsrMatrix):
            if delta.n != n:
                raise ShapeError("make_problem: delta shape does not match diagonal")
            prob.delta_kind = N.DPT_DELTA_CSR
            if self.device:
                rp, cl = delta.rowptr, delta.cols
            else:
                rp, cl = _host(delta.rowptr, np.int64), _host(delta.cols, np.int32)
            self.keep += [rp, cl]
            prob.rowptr, prob.cols, prob.vals = _ptr(rp), _ptr(cl), self._arr(delta.vals)
            prob.nnz = int(delta.vals.shape[0])
        else:
            if tuple(delta.shape) != (n, n):
                raise ShapeError("make_problem: delta shape does not match diagonal")
            prob.delta_kind = N.DPT_DELTA_DENSE
            prob.delta = self._arr(delta)
        self.prob = prob

    def _arr(self, x):
        """Pointer to x as contiguous float64 (real path) or complex128 (complex path)."""
        if self.device and _is_torch(x):
            import torch
            x = x.to(torch.complex128 if self.cplx else torch.float64)
            if not self.cplx and x.is_complex():
                x = x.real
            x = x.contiguous()
        else:
            a = np.asarray(x)
            if self.cplx:
                x = np.ascontiguousarray(a, dtype=np.complex128)
            else:
                x = np.ascontiguousarray(np.real(a) if np.iscomplexobj(a) else a, dtype=np.float64)
        self.keep.append(x)
        return _ptr(x)

    def out(self, *shape, given=None, cplx=None):
        """Output buffer; complex-valued outputs (a, eigenvalues, z) pass cplx=True."""
        c = self.cplx if cplx is None else (cplx and self.cplx)
        if given is not None:  # caller-provided output (e.g. pinned host memory)
            if tuple(given.shape) != tuple(shape):
                raise ShapeError("output buffer has the wrong shape")
            want = (np.complex128 if c else np.float64)
            if _is_torch(given):
                if not given.is_contiguous() or given.is_complex() != c:
                    raise ValueError("output tensor must be contiguous with the problem's dtype")
            elif not (given.dtype == want and given.flags["C_CONTIGUOUS"]):
                raise ValueError(f"output array must be C-contiguous {np.dtype(want).name}")
            self.keep.append(given)
            return given, _ptr(given)
        if self.device:
            import torch
            t = torch.empty(shape, dtype=torch.complex128 if c else torch.float64, device=self.keep[0].device)
            self.keep.append(t)
            return t, t.data_ptr()
        a = np.empty(shape, dtype=np.complex128 if c else np.float64)
        return a, a.ctypes.data

    def inp(self, x, *shape):
        if self.device:
            import torch
            if not (_is_torch(x) and x.is_cuda):
                x = torch.as_tensor(np.asarray(x), device=self.keep[0].device)
            x = x.to(torch.complex128 if self.cplx else torch.float64).contiguous()
            self.keep.append(x)
            return x.data_ptr()
        a = np.asarray(x)
        a = np.ascontiguousarray(a, dtype=np.complex128) if self.cplx else np.ascontiguousarray(
            np.real(a) if np.iscomplexobj(a) else a, dtype=np.float64)
        if a.shape != tuple(shape):
            raise ShapeError("dimension mismatch")
        self.keep.append(a)
        return a.ctypes.data

    def result(self, x):
        """Complex-dtype callers get complex outputs even on the real path."""
        if self.cdtype and not self.cplx and not _is_torch(x):
            return x.astype(np.complex128)
        return x

    @property
    def mem(self):
        return N.DPT_MEM_DEVICE if self.device else N.DPT_MEM_HOST


def _trace_cb(trace):
    if trace is None:
        return N.TRACE_FN(0), None
    box = {}

    def cb(k, s, r, user):
        try:
            trace(int(k), float(s), float(r))
            return 0
        except BaseException as e:  # the reference propagates the sink's exception
            box["exc"] = e
            return 1
    return N.TRACE_FN(cb), box


def _opts(o: Optional[IterationOptions]) -> N.dpt_options:
    return (o or IterationOptions())._c()


# ------------------------------------------------------------------ API ----
def _full(p, opts, trace, ramped, alpha, ctx, out=None):
    ctx = ctx or default_context()
    m = _Marshal(p)
    n = m.n
    oa, oe, orr = out if out is not None else (None, None, None)
    a, ap = m.out(n, n, given=oa)
    eig, ep = m.out(n, given=oe)
    res, rp = m.out(n, given=orr, cplx=False)
    rep, err = N.dpt_report(), N.dpt_error_info()
    cb, box = _trace_cb(trace)
    o = _opts(opts)
    if ramped:
        rc = N.lib().dpt_iterate_ramped(ctx.handle, ctypes.byref(m.prob), float(alpha), ctypes.byref(o), cb,
                                        None, ap, ep, rp, m.mem, ctypes.byref(rep), ctypes.byref(err))
    else:
        rc = N.lib().dpt_iterate_full(ctx.handle, ctypes.byref(m.prob), ctypes.byref(o), cb, None, ap, ep,
                                      rp, m.mem, ctypes.byref(rep), ctypes.byref(err))
    if rc == N.DPT_ERR_TRACE and box and "exc" in box:
        raise box["exc"]
    _raise(rc, err)
    return ConvergenceReport(EigenIterate(m.result(a), rep.iterations), m.result(eig), ConvergenceStatus(rep.status),
                             rep.iterations, res, rep.step_norm, rep.device_ms)


def iterate_full(p: PartitionedProblem, opts: Optional[IterationOptions] = None,
                 trace: Optional[Callable[[int, float, float], None]] = None, ctx: Context = None, out=None):
    """Fixed-point iteration of the full map from A = I (dpt.hpp:74-83).
    out=(a, eigenvalues, residuals) writes into caller buffers (e.g. pinned)."""
    return _full(p, opts, trace, False, 0.0, ctx, out)


def homotopy_solve(p: PartitionedProblem, stages: int, opts: Optional[IterationOptions] = None,
                   ctx: Context = None):
    """Staged continuation (dpt.hpp:145-152, dpt.cpp:505-556) on the device:
    `stages` solves along lambda s / stages, each on the problem rebased by the
    converged bases.  Report as iterate_full (iterations summed over stages)."""
    ctx = ctx or default_context()
    m = _Marshal(p)
    n = m.n
    a, ap = m.out(n, n)
    eig, ep = m.out(n)
    res, rp = m.out(n, cplx=False)
    rep, err = N.dpt_report(), N.dpt_error_info()
    _raise(N.lib().dpt_homotopy_solve(ctx.handle, ctypes.byref(m.prob), int(stages), ctypes.byref(_opts(opts)), ap,
                                      ep, rp, m.mem, ctypes.byref(rep), ctypes.byref(err)), err)
    return ConvergenceReport(EigenIterate(m.result(a), rep.iterations), m.result(eig), ConvergenceStatus(rep.status),
                             rep.iterations, res, rep.step_norm, rep.device_ms)


def _dense_host(x):
    x = np.asarray(x)
    cplx = np.iscomplexobj(x)
    return np.ascontiguousarray(x, dtype=np.complex128 if cplx else np.float64), cplx


def matmul_dense(a, b, ctx: Context = None) -> np.ndarray:
    """matmul(DenseMatrix, DenseMatrix) (matrix.cpp:130-143) on the device DMMA
    GEMM: a (m x k) @ b (k x n), real or complex host arrays."""
    ctx = ctx or default_context()
    a, ca = _dense_host(a)
    b, cb = _dense_host(b)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise ShapeError("matmul shape mismatch")
    cplx = ca or cb
    if cplx:
        a, b = a.astype(np.complex128), b.astype(np.complex128)
    c = np.zeros((a.shape[0], b.shape[1]), dtype=np.complex128 if cplx else np.float64)
    err = N.dpt_error_info()
    _raise(N.lib().dpt_matmul_dense(ctx.handle, a.shape[0], a.shape[1], b.shape[1], int(cplx), a.ctypes.data,
                                    b.ctypes.data, c.ctypes.data, N.DPT_MEM_HOST, ctypes.byref(err)), err)
    return c


def solve_linear_multi(a, b, ctx: Context = None) -> np.ndarray:
    """solve_linear_multi (matrix.cpp:519-533) on the device: a^-1 b by LU with
    partial pivoting (cluster panels + DMMA updates).  Raises RuntimeError
    ("solve_linear: singular matrix") on an exactly-zero pivot, as the reference."""
    ctx = ctx or default_context()
    a, ca = _dense_host(a)
    b, cb = _dense_host(b)
    if a.ndim != 2 or a.shape[0] != a.shape[1] or b.ndim != 2 or b.shape[0] != a.shape[0]:
        raise ShapeError("solve_linear_multi shape mismatch")
    cplx = ca or cb
    if cplx:
        a, b = a.astype(np.complex128), b.astype(np.complex128)
    x = np.zeros(b.shape, dtype=np.complex128 if cplx else np.float64)
    err = N.dpt_error_info()
    rc = N.lib().dpt_solve_linear_multi(ctx.handle, a.shape[0], b.shape[1], int(cplx), a.ctypes.data, b.ctypes.data,
                                        x.ctypes.data, N.DPT_MEM_HOST, ctypes.byref(err))
    if rc == N.DPT_ERR_UNSUPPORTED and b"singular" in err.message:
        raise RuntimeError(err.message.decode())
    _raise(rc, err)
    return x


def iterate_ramped(p: PartitionedProblem, alpha: float, opts: Optional[IterationOptions] = None,
                   trace=None, ctx: Context = None):
    """lambda_k = lambda (1 - alpha^(k-1)) (dpt.hpp:85-92); alpha in [0, 1)."""
    return _full(p, opts, trace, True, alpha, ctx)


def iterate_fixed(p: PartitionedProblem, k: int, lam, ctx: Context = None):
    """Exactly k applications of the map from I at lam (dpt.hpp:94-96)."""
    ctx = ctx or default_context()
    m = _Marshal(p, extra_complex=bool(np.iscomplexobj(np.asarray(lam)) and np.imag(lam) != 0))
    a, ap = m.out(m.n, m.n)
    rep, err = N.dpt_report(), N.dpt_error_info()
    _raise(N.lib().dpt_iterate_fixed_c(ctx.handle, ctypes.byref(m.prob), int(k), float(np.real(lam)),
                                       float(np.imag(lam)), ap, m.mem, ctypes.byref(rep), ctypes.byref(err)), err)
    return m.result(a)


def step_full(a, p: PartitionedProblem, lam, ctx: Context = None, theta=None):
    """One application of the full map to `a` (dpt.hpp:51-57).  theta: optional
    explicit gap matrix (the reference's GapMatrix); default 1/(d_i - d_j)."""
    ctx = ctx or default_context()
    cx = bool(np.iscomplexobj(np.asarray(lam)) and np.imag(lam) != 0) or _has_imag(a) or (
        theta is not None and _has_imag(theta))
    m = _Marshal(p, extra_complex=cx)
    ip = m.inp(a, m.n, m.n)
    gp = m.inp(theta, m.n, m.n) if theta is not None else None
    out, op = m.out(m.n, m.n)
    err = N.dpt_error_info()
    if gp is not None:
        rc = N.lib().dpt_step_full_gap_c(ctx.handle, ctypes.byref(m.prob), ip, gp, float(np.real(lam)),
                                         float(np.imag(lam)), op, m.mem, ctypes.byref(err))
    else:
        rc = N.lib().dpt_step_full(ctx.handle, ctypes.byref(m.prob), ip, float(np.real(lam)), op, m.mem,
                                   ctypes.byref(err)) if not m.cplx else N.lib().dpt_step_full_gap_c(
            ctx.handle, ctypes.byref(m.prob), ip, m.inp(_gap_matrix(p.d), m.n, m.n), float(np.real(lam)),
            float(np.imag(lam)), op, m.mem, ctypes.byref(err))
    _raise(rc, err)
    return m.result(out)


def _gap_matrix(d):
    """build_theta's table 1/(d_i - d_j) (zero diagonal) on the host -- only used
    to feed step_full's complex-lambda path when the caller passes no GapMatrix."""
    d = np.asarray(d.cpu().numpy() if _is_torch(d) else d, dtype=np.complex128)
    with np.errstate(divide="ignore", invalid="ignore"):
        g = 1.0 / (d[:, None] - d[None, :])
    np.fill_diagonal(g, 0.0)
    return g


def iterate_single(p: PartitionedProblem, row: int, opts: Optional[IterationOptions] = None,
                   ramp_alpha: float = 0.0, trace=None, ctx: Context = None):
    """Row-map iteration from z = e_row (dpt.hpp:107-111)."""
    ctx = ctx or default_context()
    m = _Marshal(p)
    z, zp = m.out(m.n)
    rep, err = N.dpt_report(), N.dpt_error_info()
    cb, box = _trace_cb(trace)
    o = _opts(opts)
    rc = N.lib().dpt_iterate_single(ctx.handle, ctypes.byref(m.prob), int(row), ctypes.byref(o),
                                    float(ramp_alpha), cb, None, zp, m.mem, ctypes.byref(rep),
                                    ctypes.byref(err))
    if rc == N.DPT_ERR_TRACE and box and "exc" in box:
        raise box["exc"]
    _raise(rc, err)
    eig = complex(rep.eigenvalue, rep.eigenvalue_im) if m.cdtype else rep.eigenvalue
    return SingleRowReport(m.result(z), eig, ConvergenceStatus(rep.status), rep.iterations, rep.residual,
                           rep.step_norm, rep.device_ms)


def dominant_eigenpair(p: PartitionedProblem, opts: Optional[IterationOptions] = None, ctx: Context = None):
    """Eigenvector continued from the largest level (dpt.hpp:124-129)."""
    ctx = ctx or default_context()
    m = _Marshal(p)
    zc, zcp = m.out(m.n)
    zu, zup = m.out(m.n)
    rep, err = N.dpt_report(), N.dpt_error_info()
    o = _opts(opts)
    _raise(N.lib().dpt_dominant_eigenpair(ctx.handle, ctypes.byref(m.prob), ctypes.byref(o), zcp, zup,
                                          m.mem, ctypes.byref(rep), ctypes.byref(err)), err)
    eig = complex(rep.eigenvalue, rep.eigenvalue_im) if m.cdtype else rep.eigenvalue
    return DominantEigenpair(int(rep.row), m.result(zc), m.result(zu), eig, ConvergenceStatus(rep.status),
                             rep.iterations, rep.residual, rep.step_norm, rep.device_ms)


def step_single(z, row: int, p: PartitionedProblem, lam, ctx: Context = None, gap_row=None):
    """One row-map application for chart index row (dpt.hpp:59-66)."""
    ctx = ctx or default_context()
    cx = bool(np.iscomplexobj(np.asarray(lam)) and np.imag(lam) != 0) or _has_imag(z)
    m = _Marshal(p, extra_complex=cx)
    ip = m.inp(z, m.n)
    out, op = m.out(m.n)
    err = N.dpt_error_info()
    if gap_row is None and m.cplx:
        gap_row = _gap_matrix(p.d)[int(row)]
    if gap_row is not None:
        gp = m.inp(gap_row, m.n)
        rc = N.lib().dpt_step_single_gap_c(ctx.handle, ctypes.byref(m.prob), ip, int(row), gp, float(np.real(lam)),
                                           float(np.imag(lam)), op, m.mem, ctypes.byref(err))
    else:
        rc = N.lib().dpt_step_single(ctx.handle, ctypes.byref(m.prob), ip, int(row), float(np.real(lam)), op,
                                     m.mem, ctypes.byref(err))
    _raise(rc, err)
    return m.result(out)


def eigenvalue_of(z, row: int, p: PartitionedProblem, lam, ctx: Context = None):
    """eps_row + lam (Delta z)_row (dpt.hpp:68-72)."""
    ctx = ctx or default_context()
    cx = bool(np.iscomplexobj(np.asarray(lam)) and np.imag(lam) != 0) or _has_imag(z)
    m = _Marshal(p, extra_complex=cx)
    ip = m.inp(z, m.n)
    out = (ctypes.c_double * 2)()
    err = N.dpt_error_info()
    _raise(N.lib().dpt_eigenvalue_of_c(ctx.handle, ctypes.byref(m.prob), ip, int(row), float(np.real(lam)),
                                       float(np.imag(lam)), out, m.mem, ctypes.byref(err)), err)
    return complex(out[0], out[1]) if (m.cdtype or m.cplx) else out[0]


class Plan:
    """A problem kept resident in HBM with its workspace (dpt_plan_*): repeated
    fixed-step runs of the full map (single=False) or the row map for `row`.
    The coupling is p.lam (complex problems: Re lam overridable by `lam`)."""

    def __init__(self, p: PartitionedProblem, lam: float = None, single: bool = False, row: int = 0,
                 ctx: Context = None):
        self.ctx = ctx or default_context()
        self._m = _Marshal(p)
        self.n = self._m.n
        self.single = single
        h, err = ctypes.c_void_p(), N.dpt_error_info()
        _raise(N.lib().dpt_plan_create(self.ctx.handle, ctypes.byref(self._m.prob), int(single), int(row),
                                       float(np.real(p.lam if lam is None else lam)), ctypes.byref(h),
                                       ctypes.byref(err)), err)
        self.handle = h

    def begin(self):
        err = N.dpt_error_info()
        _raise(N.lib().dpt_plan_begin(self.handle, ctypes.byref(err)), err)

    def steps(self, k: int, time_kernel: bool = False):
        """Enqueue k map applications; with time_kernel, return the summed step-kernel ms."""
        err = N.dpt_error_info()
        ms = ctypes.c_double(0.0)
        _raise(N.lib().dpt_plan_steps(self.handle, int(k), ctypes.byref(ms) if time_kernel else None,
                                      ctypes.byref(err)), err)
        return ms.value if time_kernel else None

    def read(self):
        shape = (self.n,) if self.single else (self.n, self.n)
        out = np.empty(shape, dtype=np.complex128 if self._m.cplx else np.float64)
        err = N.dpt_error_info()
        _raise(N.lib().dpt_plan_read(self.handle, out.ctypes.data, N.DPT_MEM_HOST, ctypes.byref(err)), err)
        return out

    def stats(self):
        out = np.empty(4)
        err = N.dpt_error_info()
        _raise(N.lib().dpt_plan_stats(self.handle, out.ctypes.data, ctypes.byref(err)), err)
        return out

    def close(self):
        if getattr(self, "handle", None):
            N.lib().dpt_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fp64_peak_tflops(device: int = 0) -> float:
    """Measured DMMA (FP64 tensor core) throughput of the device, TFLOP/s."""
    v, err = ctypes.c_double(0.0), N.dpt_error_info()
    _raise(N.lib().dpt_probe_fp64_peak(int(device), ctypes.byref(v), ctypes.byref(err)), err)
    return v.value


# ------------------------------------------------------------ host helpers ----
def check_degenerate(d, tol: float = 1e-12):
    """build_theta's degeneracy policy: None or the reference's first (i, j)."""
    d = _host(d, np.float64)
    i, j = ctypes.c_int64(), ctypes.c_int64()
    hit = N.lib().dpt_check_degenerate(int(d.shape[0]), d.ctypes.data, float(tol), ctypes.byref(i),
                                       ctypes.byref(j))
    return (i.value, j.value) if hit else None


def spectral_spread(d) -> float:
    d = _host(d, np.float64)
    return float(N.lib().dpt_spectral_spread(int(d.shape[0]), d.ctypes.data))


def effective_window(requested: int, n: int) -> int:
    return int(N.lib().dpt_effective_window(int(requested), int(n)))


# ------------------------------------------------------------- scan_domain ----
class CellClass(enum.IntEnum):
    """proj/include/dynspec/analysis.hpp:33-37"""
    Converged = 0
    BoundedNonConverged = 1
    Diverged = 2


@dataclass
class ScanGrid:
    """proj/include/dynspec/analysis.hpp:20-27"""
    re_min: float = -1.0
    re_max: float = 1.0
    im_min: float = -1.0
    im_max: float = 1.0
    res_re: int = 100
    res_im: int = 100


@dataclass
class ScanMode:
    """proj/include/dynspec/analysis.hpp:56-61: Full or SingleRow (kind), chart row, ramp alpha."""
    kind: str = "Full"
    row: int = 0
    ramp_alpha: float = 0.0


def grid_coordinate(lo: float, hi: float, res: int, i: int) -> float:
    """analysis.cpp:42-46"""
    if res == 0:
        raise ShapeError("grid_coordinate: empty axis")
    if res == 1:
        return 0.5 * (lo + hi)
    return lo + (hi - lo) * (float(i) / float(res - 1))


@dataclass
class DomainGrid:
    """analysis.hpp:39-54: classes / iterations are row-major with the
    imaginary index major, shape (res_im, res_re)."""
    grid: ScanGrid
    classes: np.ndarray
    iterations: np.ndarray

    def re_at(self, j: int) -> float:
        return grid_coordinate(self.grid.re_min, self.grid.re_max, self.grid.res_re, j)

    def im_at(self, i: int) -> float:
        return grid_coordinate(self.grid.im_min, self.grid.im_max, self.grid.res_im, i)


def scan_domain(base: PartitionedProblem, grid: ScanGrid, mode: ScanMode = None, opts: IterationOptions = None,
                threads: int = 0, ctx: Context = None) -> DomainGrid:
    """scan_domain (proj/src/analysis.cpp:68-138): classify every lambda cell.
    Batched on the device (one warp per cell) for small problems; `threads` is
    accepted for signature parity and ignored (the output is thread-independent
    in the reference too)."""
    mode = mode or ScanMode()
    ctx = ctx or default_context()
    m = _Marshal(base)  # the base lambda is ignored (each cell sets its own)
    g = N.dpt_scan_grid(float(grid.re_min), float(grid.re_max), float(grid.im_min), float(grid.im_max),
                        int(grid.res_re), int(grid.res_im))
    cells = int(grid.res_re) * int(grid.res_im)
    cls = np.zeros(max(cells, 0), dtype=np.uint8)
    its = np.zeros(max(cells, 0), dtype=np.int32)
    err = N.dpt_error_info()
    kind = N.DPT_SCAN_SINGLE_ROW if mode.kind == "SingleRow" else N.DPT_SCAN_FULL
    _raise(N.lib().dpt_scan_domain(ctx.handle, ctypes.byref(m.prob), ctypes.byref(g), kind, int(mode.row),
                                   float(mode.ramp_alpha), ctypes.byref(_opts(opts)), cls.ctypes.data,
                                   its.ctypes.data, ctypes.byref(err)), err)
    shape = (int(grid.res_im), int(grid.res_re))
    return DomainGrid(grid, cls.reshape(shape), its.reshape(shape))


# ----------------------------------------------------------- Matrix Market ----
def read_matrix_market(path: str, threads: int = 0):
    """read_matrix_market (proj/src/matrix_market.cpp:70-143): a CsrMatrix for
    coordinate files, a dense row-major ndarray for array files; complex dtype
    for the complex field.  Bit-identical to the reference; parsed with
    `threads` host threads (0 = all).  Raises IoError like the reference."""
    m = N.dpt_mm_matrix()
    err = N.dpt_error_info()
    _raise(N.lib().dpt_mm_read(str(path).encode(), int(threads), ctypes.byref(m), ctypes.byref(err)), err)
    try:
        cx = 2 if m.is_complex else 1
        nval = int(m.nnz) * cx

        def arr(ptr, count, ctype, dtype):
            if count == 0:
                return np.zeros(0, dtype=dtype)
            return np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctype)), shape=(count,)).astype(dtype, copy=True)

        vals = arr(m.vals, nval, ctypes.c_double, np.float64)
        if m.is_complex:
            vals = vals.view(np.complex128)
        if not m.is_sparse:
            return vals.reshape(int(m.rows), int(m.cols))
        rp = arr(m.rowptr, int(m.rows) + 1, ctypes.c_int64, np.int64)
        ci = arr(m.colidx, int(m.nnz), ctypes.c_int64, np.int64)
        cols = ci.astype(np.int32) if int(m.cols) < 2 ** 31 else ci
        if int(m.rows) != int(m.cols):
            return CsrMatrix(int(m.rows), rp, cols, vals, ncols=int(m.cols))
        return CsrMatrix(int(m.rows), rp, cols, vals)
    finally:
        N.lib().dpt_mm_free(ctypes.byref(m))


def write_matrix_market(m, path: str, threads: int = 0) -> None:
    """write_matrix_market (matrix_market.cpp:170-195): array format for dense,
    coordinate for CSR, real field when every imaginary part is 0, "%.17g"."""
    err = N.dpt_error_info()
    if isinstance(m, CsrMatrix):
        vals = np.asarray(m.vals)
        cplx = np.iscomplexobj(vals)
        vals = np.ascontiguousarray(vals, dtype=np.complex128 if cplx else np.float64)
        rp = np.ascontiguousarray(m.rowptr, dtype=np.int64)
        ci = np.ascontiguousarray(m.cols, dtype=np.int64)
        ncols = getattr(m, "ncols", None) or m.n
        _raise(N.lib().dpt_mm_write_csr(str(path).encode(), int(m.n), int(ncols), rp.ctypes.data, ci.ctypes.data,
                                        vals.ctypes.data, int(cplx), int(threads), ctypes.byref(err)), err)
        return
    a = np.asarray(m)
    if a.ndim != 2:
        raise ShapeError("write_matrix_market: dense matrix must be 2-D")
    cplx = np.iscomplexobj(a)
    a = np.ascontiguousarray(a, dtype=np.complex128 if cplx else np.float64)
    _raise(N.lib().dpt_mm_write_dense(str(path).encode(), int(a.shape[0]), int(a.shape[1]), a.ctypes.data, int(cplx),
                                      int(threads), ctypes.byref(err)), err)
