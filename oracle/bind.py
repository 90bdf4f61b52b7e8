"""TEST INFRASTRUCTURE ONLY -- ctypes access to the two CPU checkers:

  restatement  oracle/libdpt_oracle.so     (dpt_oracle.c, the C restatement)
  reference    oracle/_ref/libdynspec_ref.so (the reference's own sources + ref_capi.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this module.  The product (paper_2002_12872_b200) never does.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, Structure, c_double, c_int, c_int32, c_int64, c_void_p
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libdpt_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdynspec_ref.so")

ORC_DENSE, ORC_CSR = 0, 1
STATUS = ["Converged", "BoundedNonConverged", "Diverged", "MaxIterations"]
ORC_OK, ORC_ERR_SHAPE, ORC_ERR_DEGENERATE, ORC_ERR_INVALID = 0, 1, 2, 3


class orc_problem(Structure):
    _fields_ = [("n", c_int64), ("d", c_void_p), ("kind", c_int), ("delta", c_void_p),
                ("rowptr", c_void_p), ("cols", c_void_p), ("vals", c_void_p), ("lambda_", c_double)]


class orc_options(Structure):
    _fields_ = [("tol", c_double), ("residual_tol", c_double), ("max_iter", c_int),
                ("divergence_threshold", c_double), ("cycle_window", c_int), ("degeneracy_tol", c_double)]


class orc_report(Structure):
    _fields_ = [("status", c_int), ("iterations", c_int), ("step_norm", c_double),
                ("degenerate_i", c_int64), ("degenerate_j", c_int64)]


class orc_single_report(Structure):
    _fields_ = [("status", c_int), ("iterations", c_int), ("step_norm", c_double), ("eigenvalue", c_double),
                ("residual", c_double), ("degenerate_i", c_int64), ("degenerate_j", c_int64)]


@dataclass
class FullResult:
    rc: int
    status: int
    iterations: int
    step_norm: float
    a: np.ndarray
    eig: np.ndarray
    res: np.ndarray
    trace_step: np.ndarray = None
    trace_res: np.ndarray = None
    degenerate: tuple = None
    imag_max: float = 0.0


@dataclass
class SingleResult:
    rc: int
    status: int
    iterations: int
    step_norm: float
    eigenvalue: float
    residual: float
    z: np.ndarray
    z_unit: np.ndarray = None
    row: int = -1
    trace_step: np.ndarray = None
    trace_res: np.ndarray = None
    degenerate: tuple = None


def _load(path, prefix):
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built (make -C oracle)")
    L = ctypes.CDLL(path)
    P = POINTER
    getattr(L, prefix + "iterate_full").argtypes = (
        [P(orc_problem), P(orc_options), c_int, c_double, c_void_p, c_void_p, c_void_p, P(orc_report),
         c_void_p, c_void_p] + ([c_void_p] if prefix == "ref_" else []))
    getattr(L, prefix + "iterate_fixed").argtypes = [P(orc_problem), c_int, c_double, c_void_p]
    getattr(L, prefix + "step_full").argtypes = [P(orc_problem), c_void_p, c_double, c_void_p]
    getattr(L, prefix + "iterate_single").argtypes = [P(orc_problem), c_int64, P(orc_options), c_double,
                                                      c_void_p, P(orc_single_report), c_void_p, c_void_p]
    getattr(L, prefix + "dominant_eigenpair").argtypes = [P(orc_problem), P(orc_options), c_void_p, c_void_p,
                                                          P(orc_single_report), P(c_int64)]
    getattr(L, prefix + "step_single").argtypes = [P(orc_problem), c_void_p, c_int64, c_double, c_void_p]
    getattr(L, prefix + "eigenvalue_of").argtypes = [P(orc_problem), c_void_p, c_int64, c_double, P(c_double)]
    getattr(L, prefix + "step_rows").argtypes = [P(orc_problem), c_int64, c_int64, c_void_p, c_double, c_void_p]
    if prefix == "ref_":
        L.ref_check_degenerate.argtypes = [c_int64, c_void_p, c_double, P(c_int64), P(c_int64)]
        L.ref_prepare.argtypes = [P(orc_problem)]
        L.ref_prepare.restype = c_void_p
        L.ref_release.argtypes = [c_void_p]
        L.ref_prepared_step_rows.argtypes = [c_void_p, c_int64, c_int64, c_void_p, c_double, c_void_p]
    else:
        L.orc_check_degenerate.argtypes = [c_int64, c_void_p, c_double, P(c_int64), P(c_int64)]
        L.orc_effective_window.argtypes = [c_int, c_int64]
    return L


class Checker:
    """One CPU implementation of the path: 'oracle' (restatement) or 'reference'."""

    def __init__(self, which: str = "oracle"):
        self.which = which
        self.prefix = "ref_" if which == "reference" else "orc_"
        self.L = _load(REF_SO if which == "reference" else ORACLE_SO, self.prefix)

    def _fn(self, name):
        return getattr(self.L, self.prefix + name)

    @staticmethod
    def _prob(p):
        """p: paper_2002_12872_b200.PartitionedProblem with numpy parts."""
        keep = []
        d = np.ascontiguousarray(p.d, dtype=np.float64)
        keep.append(d)
        pr = orc_problem()
        pr.n = d.shape[0]
        pr.d = d.ctypes.data
        pr.lambda_ = float(p.lam)
        if hasattr(p.delta, "rowptr"):
            rp = np.ascontiguousarray(p.delta.rowptr, dtype=np.int64)
            cl = np.ascontiguousarray(p.delta.cols, dtype=np.int32)
            vl = np.ascontiguousarray(p.delta.vals, dtype=np.float64)
            keep += [rp, cl, vl]
            pr.kind = ORC_CSR
            pr.rowptr, pr.cols, pr.vals = rp.ctypes.data, cl.ctypes.data, vl.ctypes.data
        else:
            a = np.ascontiguousarray(p.delta, dtype=np.float64)
            keep.append(a)
            pr.kind = ORC_DENSE
            pr.delta = a.ctypes.data
        return pr, keep

    @staticmethod
    def _opts(o: dict):
        base = dict(tol=1e-12, residual_tol=1e-10, max_iter=10000, divergence_threshold=1e8, cycle_window=16,
                    degeneracy_tol=1e-12)
        base.update(o or {})
        return orc_options(base["tol"], base["residual_tol"], int(base["max_iter"]), base["divergence_threshold"],
                           int(base["cycle_window"]), base["degeneracy_tol"])

    def iterate_full(self, p, opts=None, trace=False, ramped=False, alpha=0.0) -> FullResult:
        pr, keep = self._prob(p)
        n = pr.n
        o = self._opts(opts)
        a = np.zeros((n, n))
        eig = np.zeros(n)
        res = np.zeros(n)
        rep = orc_report()
        cap = max(o.max_iter, 1) + 1
        ts = np.full(cap, np.nan) if trace else None
        tr = np.full(cap, np.nan) if trace else None
        args = [ctypes.byref(pr), ctypes.byref(o), int(ramped), float(alpha), a.ctypes.data, eig.ctypes.data,
                res.ctypes.data, ctypes.byref(rep), ts.ctypes.data if trace else None,
                tr.ctypes.data if trace else None]
        im = ctypes.c_double(0.0)
        if self.prefix == "ref_":
            args.append(ctypes.addressof(im))
        rc = self._fn("iterate_full")(*args)
        k = rep.iterations if trace else 0
        return FullResult(rc, rep.status, rep.iterations, rep.step_norm, a, eig, res,
                          ts[:k] if trace else None, tr[:k] if trace else None,
                          (rep.degenerate_i, rep.degenerate_j) if rc == ORC_ERR_DEGENERATE else None, im.value)

    def iterate_fixed(self, p, k, lam):
        pr, keep = self._prob(p)
        a = np.zeros((pr.n, pr.n))
        rc = self._fn("iterate_fixed")(ctypes.byref(pr), int(k), float(lam), a.ctypes.data)
        return rc, a

    def step_full(self, a, p, lam):
        pr, keep = self._prob(p)
        a = np.ascontiguousarray(a, dtype=np.float64)
        out = np.zeros_like(a)
        self._fn("step_full")(ctypes.byref(pr), a.ctypes.data, float(lam), out.ctypes.data)
        return out

    def step_rows(self, p, row0, a_rows, lam):
        pr, keep = self._prob(p)
        a_rows = np.ascontiguousarray(a_rows, dtype=np.float64)
        out = np.zeros_like(a_rows)
        self._fn("step_rows")(ctypes.byref(pr), int(row0), int(a_rows.shape[0]), a_rows.ctypes.data, float(lam),
                              out.ctypes.data)
        return out

    def iterate_single(self, p, row, opts=None, ramp_alpha=0.0, trace=False) -> SingleResult:
        pr, keep = self._prob(p)
        o = self._opts(opts)
        z = np.zeros(pr.n)
        rep = orc_single_report()
        cap = max(o.max_iter, 1) + 1
        ts = np.full(cap, np.nan) if trace else None
        tr = np.full(cap, np.nan) if trace else None
        rc = self._fn("iterate_single")(ctypes.byref(pr), int(row), ctypes.byref(o), float(ramp_alpha),
                                        z.ctypes.data, ctypes.byref(rep), ts.ctypes.data if trace else None,
                                        tr.ctypes.data if trace else None)
        k = rep.iterations if trace else 0
        return SingleResult(rc, rep.status, rep.iterations, rep.step_norm, rep.eigenvalue, rep.residual, z,
                            trace_step=ts[:k] if trace else None, trace_res=tr[:k] if trace else None,
                            degenerate=(rep.degenerate_i, rep.degenerate_j) if rc == ORC_ERR_DEGENERATE else None)

    def dominant_eigenpair(self, p, opts=None) -> SingleResult:
        pr, keep = self._prob(p)
        o = self._opts(opts)
        zc = np.zeros(pr.n)
        zu = np.zeros(pr.n)
        rep = orc_single_report()
        row = ctypes.c_int64(-1)
        rc = self._fn("dominant_eigenpair")(ctypes.byref(pr), ctypes.byref(o), zc.ctypes.data, zu.ctypes.data,
                                            ctypes.byref(rep), ctypes.byref(row))
        return SingleResult(rc, rep.status, rep.iterations, rep.step_norm, rep.eigenvalue, rep.residual, zc, zu,
                            row.value,
                            degenerate=(rep.degenerate_i, rep.degenerate_j) if rc == ORC_ERR_DEGENERATE else None)

    def step_single(self, z, row, p, lam):
        pr, keep = self._prob(p)
        z = np.ascontiguousarray(z, dtype=np.float64)
        out = np.zeros_like(z)
        self._fn("step_single")(ctypes.byref(pr), z.ctypes.data, int(row), float(lam), out.ctypes.data)
        return out

    def eigenvalue_of(self, z, row, p, lam):
        pr, keep = self._prob(p)
        z = np.ascontiguousarray(z, dtype=np.float64)
        out = ctypes.c_double()
        self._fn("eigenvalue_of")(ctypes.byref(pr), z.ctypes.data, int(row), float(lam), ctypes.byref(out))
        return out.value

    def check_degenerate(self, d, tol=1e-12):
        d = np.ascontiguousarray(d, dtype=np.float64)
        i, j = ctypes.c_int64(), ctypes.c_int64()
        hit = self._fn("check_degenerate")(d.shape[0], d.ctypes.data, float(tol), ctypes.byref(i), ctypes.byref(j))
        return (i.value, j.value) if hit else None


def available(which: str) -> bool:
    return os.path.exists(REF_SO if which == "reference" else ORACLE_SO)


# ---- complex inputs: the reference library's native std::complex<double> path ----
class orc_cproblem(Structure):
    _fields_ = [("n", c_int64), ("d", c_void_p), ("kind", c_int), ("delta", c_void_p), ("rowptr", c_void_p),
                ("cols", c_void_p), ("vals", c_void_p), ("lam_re", c_double), ("lam_im", c_double)]


class ComplexReference:
    """The reference (oracle/_ref) on complex problems: results as complex128 numpy arrays."""

    def __init__(self):
        L = ctypes.CDLL(REF_SO)
        P = POINTER
        L.ref_c_iterate_full.argtypes = [P(orc_cproblem), P(orc_options), c_int, c_double, c_void_p, c_void_p,
                                         c_void_p, P(orc_report), c_void_p, c_void_p]
        L.ref_c_iterate_single.argtypes = [P(orc_cproblem), c_int64, P(orc_options), c_double, c_void_p, c_void_p,
                                           P(orc_single_report)]
        L.ref_c_dominant.argtypes = [P(orc_cproblem), P(orc_options), c_void_p, c_void_p, c_void_p,
                                     P(orc_single_report), P(c_int64)]
        L.ref_c_iterate_fixed.argtypes = [P(orc_cproblem), c_int, c_double, c_double, c_void_p]
        L.ref_c_step_full.argtypes = [P(orc_cproblem), c_void_p, c_double, c_double, c_void_p]
        L.ref_c_step_single.argtypes = [P(orc_cproblem), c_void_p, c_int64, c_double, c_double, c_void_p, c_void_p]
        L.ref_c_check_degenerate.argtypes = [c_int64, c_void_p, c_double, P(c_int64), P(c_int64)]
        L.ref_c_homotopy.argtypes = [P(orc_cproblem), c_int, P(orc_options), c_void_p, c_void_p, c_void_p,
                                     P(orc_report)]
        L.ref_c_matmul.argtypes = [c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p]
        L.ref_c_solve_linear_multi.argtypes = [c_int64, c_int64, c_void_p, c_void_p, c_void_p]
        L.ref_scan_domain.argtypes = [P(orc_cproblem), c_double, c_double, c_double, c_double, c_int64, c_int64, c_int,
                                      c_int64, c_double, P(orc_options), c_int, c_void_p, c_void_p, P(c_int64),
                                      P(c_int64)]
        self.L = L

    @staticmethod
    def _prob(p):
        keep = []
        d = np.ascontiguousarray(p.d, dtype=np.complex128)
        keep.append(d)
        pr = orc_cproblem()
        pr.n = d.shape[0]
        pr.d = d.ctypes.data
        pr.lam_re, pr.lam_im = float(np.real(p.lam)), float(np.imag(p.lam))
        if hasattr(p.delta, "rowptr"):
            rp = np.ascontiguousarray(p.delta.rowptr, dtype=np.int64)
            cl = np.ascontiguousarray(p.delta.cols, dtype=np.int32)
            vl = np.ascontiguousarray(p.delta.vals, dtype=np.complex128)
            keep += [rp, cl, vl]
            pr.kind = ORC_CSR
            pr.rowptr, pr.cols, pr.vals = rp.ctypes.data, cl.ctypes.data, vl.ctypes.data
        else:
            a = np.ascontiguousarray(p.delta, dtype=np.complex128)
            keep.append(a)
            pr.kind = ORC_DENSE
            pr.delta = a.ctypes.data
        return pr, keep

    def iterate_full(self, p, opts=None, ramped=False, alpha=0.0, trace=False):
        pr, keep = self._prob(p)
        n = pr.n
        o = Checker._opts(opts)
        a = np.zeros((n, n), np.complex128)
        eig = np.zeros(n, np.complex128)
        res = np.zeros(n)
        rep = orc_report()
        cap = max(o.max_iter, 1) + 1
        ts = np.full(cap, np.nan) if trace else None
        tr = np.full(cap, np.nan) if trace else None
        rc = self.L.ref_c_iterate_full(ctypes.byref(pr), ctypes.byref(o), int(ramped), float(alpha), a.ctypes.data,
                                       eig.ctypes.data, res.ctypes.data, ctypes.byref(rep),
                                       ts.ctypes.data if trace else None, tr.ctypes.data if trace else None)
        k = rep.iterations if trace else 0
        return FullResult(rc, rep.status, rep.iterations, rep.step_norm, a, eig, res,
                          ts[:k] if trace else None, tr[:k] if trace else None,
                          (rep.degenerate_i, rep.degenerate_j) if rc == ORC_ERR_DEGENERATE else None)

    def iterate_single(self, p, row, opts=None, ramp_alpha=0.0):
        pr, keep = self._prob(p)
        o = Checker._opts(opts)
        z = np.zeros(pr.n, np.complex128)
        e = np.zeros(2)
        rep = orc_single_report()
        rc = self.L.ref_c_iterate_single(ctypes.byref(pr), int(row), ctypes.byref(o), float(ramp_alpha),
                                         z.ctypes.data, e.ctypes.data, ctypes.byref(rep))
        return SingleResult(rc, rep.status, rep.iterations, rep.step_norm, complex(e[0], e[1]), rep.residual, z)

    def dominant_eigenpair(self, p, opts=None):
        pr, keep = self._prob(p)
        o = Checker._opts(opts)
        zc = np.zeros(pr.n, np.complex128)
        zu = np.zeros(pr.n, np.complex128)
        e = np.zeros(2)
        rep = orc_single_report()
        row = ctypes.c_int64(-1)
        rc = self.L.ref_c_dominant(ctypes.byref(pr), ctypes.byref(o), zc.ctypes.data, zu.ctypes.data,
                                   e.ctypes.data, ctypes.byref(rep), ctypes.byref(row))
        return SingleResult(rc, rep.status, rep.iterations, rep.step_norm, complex(e[0], e[1]), rep.residual, zc,
                            zu, row.value)

    def iterate_fixed(self, p, k, lam):
        pr, keep = self._prob(p)
        a = np.zeros((pr.n, pr.n), np.complex128)
        self.L.ref_c_iterate_fixed(ctypes.byref(pr), int(k), float(np.real(lam)), float(np.imag(lam)), a.ctypes.data)
        return a

    def step_full(self, a, p, lam):
        pr, keep = self._prob(p)
        a = np.ascontiguousarray(a, dtype=np.complex128)
        out = np.zeros_like(a)
        self.L.ref_c_step_full(ctypes.byref(pr), a.ctypes.data, float(np.real(lam)), float(np.imag(lam)),
                               out.ctypes.data)
        return out

    def step_single(self, z, row, p, lam):
        """(step_single(z), eigenvalue_of(z)) for chart row."""
        pr, keep = self._prob(p)
        z = np.ascontiguousarray(z, dtype=np.complex128)
        out = np.zeros_like(z)
        e = np.zeros(2)
        self.L.ref_c_step_single(ctypes.byref(pr), z.ctypes.data, int(row), float(np.real(lam)), float(np.imag(lam)),
                                 out.ctypes.data, e.ctypes.data)
        return out, complex(e[0], e[1])

    def check_degenerate(self, d, tol=1e-12):
        d = np.ascontiguousarray(d, dtype=np.complex128)
        i, j = ctypes.c_int64(), ctypes.c_int64()
        hit = self.L.ref_c_check_degenerate(d.shape[0], d.ctypes.data, float(tol), ctypes.byref(i), ctypes.byref(j))
        return (i.value, j.value) if hit else None

    def homotopy(self, p, stages, opts=None):
        pr, keep = self._prob(p)
        n = pr.n
        a = np.zeros((n, n), np.complex128)
        eig = np.zeros(n, np.complex128)
        res = np.zeros(n)
        rep = orc_report()
        rc = self.L.ref_c_homotopy(ctypes.byref(pr), int(stages), ctypes.byref(Checker._opts(opts)), a.ctypes.data,
                                   eig.ctypes.data, res.ctypes.data, ctypes.byref(rep))
        return FullResult(rc, rep.status, rep.iterations, rep.step_norm, a, eig, res)

    def matmul(self, a, b):
        """The reference's matmul(DenseMatrix, DenseMatrix) (matrix.cpp:130-143)."""
        a = np.ascontiguousarray(a, dtype=np.complex128)
        b = np.ascontiguousarray(b, dtype=np.complex128)
        c = np.zeros((a.shape[0], b.shape[1]), np.complex128)
        assert self.L.ref_c_matmul(a.shape[0], a.shape[1], b.shape[1], a.ctypes.data, b.ctypes.data,
                                   c.ctypes.data) == 0
        return c

    def solve_linear_multi(self, a, b):
        """The reference's solve_linear_multi (matrix.cpp:519-533): (rc, x); rc 8 = singular."""
        a = np.ascontiguousarray(a, dtype=np.complex128)
        b = np.ascontiguousarray(b, dtype=np.complex128)
        x = np.zeros(b.shape, np.complex128)
        rc = self.L.ref_c_solve_linear_multi(a.shape[0], b.shape[1], a.ctypes.data, b.ctypes.data, x.ctypes.data)
        return rc, x

    def scan_domain(self, p, grid, mode="Full", row=0, ramp_alpha=0.0, opts=None, threads=0):
        """The reference's scan_domain: (rc, classes[res_im, res_re] uint8, iterations int32, degenerate)."""
        pr, keep = self._prob(p)
        o = Checker._opts(opts)
        cells = int(grid.res_re) * int(grid.res_im)
        cls = np.zeros(max(cells, 1), np.uint8)
        its = np.zeros(max(cells, 1), np.int32)
        di, dj = ctypes.c_int64(-1), ctypes.c_int64(-1)
        rc = self.L.ref_scan_domain(ctypes.byref(pr), grid.re_min, grid.re_max, grid.im_min, grid.im_max,
                                    int(grid.res_re), int(grid.res_im), 1 if mode == "SingleRow" else 0, int(row),
                                    float(ramp_alpha), ctypes.byref(o), int(threads), cls.ctypes.data,
                                    its.ctypes.data, ctypes.byref(di), ctypes.byref(dj))
        shape = (int(grid.res_im), int(grid.res_re))
        return rc, cls[:cells].reshape(shape), its[:cells].reshape(shape), (di.value, dj.value)


class ReferenceMatrixMarket:
    """The reference's read_matrix_market / write_matrix_market (oracle/_ref)."""

    def __init__(self):
        L = ctypes.CDLL(REF_SO)
        P = POINTER
        L.ref_mm_read.argtypes = [ctypes.c_char_p, P(c_int64), P(c_int64), P(c_int), P(c_int64), P(c_void_p),
                                  ctypes.c_char_p, c_int]
        L.ref_mm_get.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p]
        L.ref_mm_release.argtypes = [c_void_p]
        L.ref_mm_write_dense.argtypes = [ctypes.c_char_p, c_int64, c_int64, c_void_p]
        L.ref_mm_write_csr.argtypes = [ctypes.c_char_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p]
        self.L = L

    def read(self, path):
        """(rc, message, result): result = ('dense', complex array) or ('csr', rowptr, colidx, complex vals)."""
        rows, cols, nnz = c_int64(), c_int64(), c_int64()
        sp = c_int()
        h = c_void_p()
        msg = ctypes.create_string_buffer(1024)
        rc = self.L.ref_mm_read(str(path).encode(), ctypes.byref(rows), ctypes.byref(cols), ctypes.byref(sp),
                                ctypes.byref(nnz), ctypes.byref(h), msg, 1024)
        if rc != 0:
            return rc, msg.value.decode(errors="replace"), None
        try:
            vals = np.zeros(2 * max(nnz.value, 1))
            if sp.value:
                rp = np.zeros(rows.value + 1, np.int64)
                ci = np.zeros(max(nnz.value, 1), np.int64)
                self.L.ref_mm_get(h, rp.ctypes.data, ci.ctypes.data, vals.ctypes.data)
                return 0, "", ("csr", rp, ci[:nnz.value], vals[:2 * nnz.value].view(np.complex128), cols.value)
            self.L.ref_mm_get(h, None, None, vals.ctypes.data)
            return 0, "", ("dense", vals[:2 * nnz.value].view(np.complex128).reshape(rows.value, cols.value))
        finally:
            self.L.ref_mm_release(h)

    def write_dense(self, a, path):
        a = np.ascontiguousarray(a, dtype=np.complex128)
        self.L.ref_mm_write_dense(str(path).encode(), a.shape[0], a.shape[1], a.ctypes.data)

    def write_csr(self, rows, cols, rp, ci, vals, path):
        rp = np.ascontiguousarray(rp, dtype=np.int64)
        ci = np.ascontiguousarray(ci, dtype=np.int64)
        vals = np.ascontiguousarray(vals, dtype=np.complex128)
        self.L.ref_mm_write_csr(str(path).encode(), rows, cols, rp.ctypes.data, ci.ctypes.data, vals.ctypes.data)
