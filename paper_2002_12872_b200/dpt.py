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
        self.i, self.j, self.ei, self.ej = int(i), int(j), float(ei), float(ej)

    def first(self):
        return self.i

    def second(self):
        return self.j


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
    """CSR with int64 row offsets, int32 sorted columns, FP64 values (matrix.hpp:73-106)."""
    n: int
    rowptr: np.ndarray
    cols: np.ndarray
    vals: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.vals.shape[0])

    def todense(self) -> np.ndarray:
        out = np.zeros((self.n, self.n))
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
        raise DegenerateSpectrum(msg, err.i, err.j, err.ei, err.ej)
    if rc in (N.DPT_ERR_INVALID_ARG, N.DPT_ERR_NON_REAL):
        raise ValueError(msg)
    if rc == N.DPT_ERR_NO_DEVICE:
        raise NoDeviceError(msg)
    if rc == N.DPT_ERR_TRACE:
        raise TraceAborted(msg)
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


class _Marshal:
    """Keeps the arrays of one call alive and builds the dpt_problem."""

    def __init__(self, p: PartitionedProblem):
        self.keep = []
        d = p.d
        self.device = _is_torch(d) and d.is_cuda
        if self.device:
            self.keep.append(d)
            dptr = d.data_ptr()
        else:
            d = _host(d, np.float64)
            if d.ndim != 1:
                raise ShapeError("make_problem: diagonal must be a vector")
            self.keep.append(d)
            dptr = d.ctypes.data
        n = int(d.shape[0])
        self.n = n
        prob = N.dpt_problem()
        prob.n = n
        prob.d = dptr
        prob.lambda_ = float(np.real(p.lam))
        if np.iscomplexobj(np.asarray(p.lam)) and np.imag(p.lam) != 0:
            raise ValueError("non-real input: the B200 path is real FP64 (complex lambda unsupported)")
        prob.mem = N.DPT_MEM_DEVICE if self.device else N.DPT_MEM_HOST
        delta = p.delta
        if isinstance(delta, CsrMatrix):
            if delta.n != n:
                raise ShapeError("make_problem: delta shape does not match diagonal")
            prob.delta_kind = N.DPT_DELTA_CSR
            if self.device:
                rp, cl, vl = delta.rowptr, delta.cols, delta.vals
            else:
                rp, cl, vl = (_host(delta.rowptr, np.int64), _host(delta.cols, np.int32),
                              _host(delta.vals, np.float64))
            self.keep += [rp, cl, vl]
            prob.rowptr, prob.cols, prob.vals = _ptr(rp), _ptr(cl), _ptr(vl)
            prob.nnz = int(vl.shape[0])
        else:
            if not self.device:
                if np.iscomplexobj(delta):
                    if np.any(np.imag(delta) != 0):
                        raise ValueError("non-real input: the B200 path is real FP64")
                    delta = np.real(delta)
                delta = _host(delta, np.float64)
            if tuple(delta.shape) != (n, n):
                raise ShapeError("make_problem: delta shape does not match diagonal")
            self.keep.append(delta)
            prob.delta_kind = N.DPT_DELTA_DENSE
            prob.delta = _ptr(delta)
        self.prob = prob

    def out(self, *shape, given=None):
        if given is not None:  # caller-provided output (e.g. pinned host memory)
            if tuple(given.shape) != tuple(shape):
                raise ShapeError("output buffer has the wrong shape")
            if _is_torch(given):
                if not given.is_contiguous() or str(given.dtype) != "torch.float64":
                    raise ValueError("output tensor must be contiguous float64")
            elif not (given.dtype == np.float64 and given.flags["C_CONTIGUOUS"]):
                raise ValueError("output array must be C-contiguous float64")
            self.keep.append(given)
            return given, _ptr(given)
        if self.device:
            import torch
            t = torch.empty(shape, dtype=torch.float64, device=self.keep[0].device)
            self.keep.append(t)
            return t, t.data_ptr()
        a = np.empty(shape, dtype=np.float64)
        return a, a.ctypes.data

    def inp(self, x, *shape):
        if self.device:
            if not (_is_torch(x) and x.is_cuda):
                import torch
                x = torch.as_tensor(np.asarray(x, dtype=np.float64), device=self.keep[0].device)
            x = x.contiguous()
            self.keep.append(x)
            return x.data_ptr()
        a = _host(x, np.float64)
        if a.shape != tuple(shape):
            raise ShapeError("dimension mismatch")
        self.keep.append(a)
        return a.ctypes.data

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
    res, rp = m.out(n, given=orr)
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
    return ConvergenceReport(EigenIterate(a, rep.iterations), eig, ConvergenceStatus(rep.status),
                             rep.iterations, res, rep.step_norm, rep.device_ms)


def iterate_full(p: PartitionedProblem, opts: Optional[IterationOptions] = None,
                 trace: Optional[Callable[[int, float, float], None]] = None, ctx: Context = None, out=None):
    """Fixed-point iteration of the full map from A = I (dpt.hpp:74-83).
    out=(a, eigenvalues, residuals) writes into caller buffers (e.g. pinned)."""
    return _full(p, opts, trace, False, 0.0, ctx, out)


def iterate_ramped(p: PartitionedProblem, alpha: float, opts: Optional[IterationOptions] = None,
                   trace=None, ctx: Context = None):
    """lambda_k = lambda (1 - alpha^(k-1)) (dpt.hpp:85-92); alpha in [0, 1)."""
    return _full(p, opts, trace, True, alpha, ctx)


def iterate_fixed(p: PartitionedProblem, k: int, lam: float, ctx: Context = None):
    """Exactly k applications of the map from I at lam (dpt.hpp:94-96)."""
    ctx = ctx or default_context()
    m = _Marshal(p)
    a, ap = m.out(m.n, m.n)
    rep, err = N.dpt_report(), N.dpt_error_info()
    _raise(N.lib().dpt_iterate_fixed(ctx.handle, ctypes.byref(m.prob), int(k), float(lam), ap, m.mem,
                                     ctypes.byref(rep), ctypes.byref(err)), err)
    return a


def step_full(a, p: PartitionedProblem, lam: float, ctx: Context = None):
    """One application of the full map to `a` (dpt.hpp:51-57)."""
    ctx = ctx or default_context()
    m = _Marshal(p)
    ip = m.inp(a, m.n, m.n)
    out, op = m.out(m.n, m.n)
    err = N.dpt_error_info()
    _raise(N.lib().dpt_step_full(ctx.handle, ctypes.byref(m.prob), ip, float(lam), op, m.mem,
                                 ctypes.byref(err)), err)
    return out


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
    return SingleRowReport(z, rep.eigenvalue, ConvergenceStatus(rep.status), rep.iterations, rep.residual,
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
    return DominantEigenpair(int(rep.row), zc, zu, rep.eigenvalue, ConvergenceStatus(rep.status),
                             rep.iterations, rep.residual, rep.step_norm, rep.device_ms)


def step_single(z, row: int, p: PartitionedProblem, lam: float, ctx: Context = None):
    """One row-map application for chart index row (dpt.hpp:59-66)."""
    ctx = ctx or default_context()
    m = _Marshal(p)
    ip = m.inp(z, m.n)
    out, op = m.out(m.n)
    err = N.dpt_error_info()
    _raise(N.lib().dpt_step_single(ctx.handle, ctypes.byref(m.prob), ip, int(row), float(lam), op, m.mem,
                                   ctypes.byref(err)), err)
    return out


def eigenvalue_of(z, row: int, p: PartitionedProblem, lam: float, ctx: Context = None) -> float:
    """eps_row + lam (Delta z)_row (dpt.hpp:68-72)."""
    ctx = ctx or default_context()
    m = _Marshal(p)
    ip = m.inp(z, m.n)
    out = ctypes.c_double()
    err = N.dpt_error_info()
    _raise(N.lib().dpt_eigenvalue_of(ctx.handle, ctypes.byref(m.prob), ip, int(row), float(lam),
                                     ctypes.byref(out), m.mem, ctypes.byref(err)), err)
    return out.value


class Plan:
    """A problem kept resident in HBM with its workspace (dpt_plan_*): repeated
    fixed-step runs of the full map (single=False) or the row map for `row`."""

    def __init__(self, p: PartitionedProblem, lam: float = None, single: bool = False, row: int = 0,
                 ctx: Context = None):
        self.ctx = ctx or default_context()
        self._m = _Marshal(p)
        self.n = self._m.n
        self.single = single
        h, err = ctypes.c_void_p(), N.dpt_error_info()
        _raise(N.lib().dpt_plan_create(self.ctx.handle, ctypes.byref(self._m.prob), int(single), int(row),
                                       float(p.lam if lam is None else lam), ctypes.byref(h),
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
        out = np.empty(shape)
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
