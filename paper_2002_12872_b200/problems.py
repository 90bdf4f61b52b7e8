"""Seeded synthetic inputs for BASELINE.json's configs, as numpy
host arrays.  The random source restates the reference's Rng
(proj/include/dynspec/rng.hpp:12-54) in csrc/problems.cpp.  These are inputs,
not solver code: tests and bench.py feed the same arrays to the reference
build, the C restatement and the CUDA path.
"""
from __future__ import annotations

import math

import numpy as np

from . import _native as N
from .dpt import CsrMatrix, PartitionedProblem


def rng_u64(seed: int, tag: str, skip: int = 0) -> int:
    return int(N.problems_lib().dpt_gen_rng_u64(seed, tag.encode(), skip))


def theta_linear(n: int, scale: float = 1.0) -> np.ndarray:
    t = np.empty(n)
    N.problems_lib().dpt_gen_theta_linear(n, scale, t.ctypes.data)
    return t


def theta_uniform_sorted(n: int, seed: int, hi: float, min_gap: float) -> np.ndarray:
    t = np.empty(n)
    if N.problems_lib().dpt_gen_theta_uniform_sorted(n, seed, hi, min_gap, t.ctypes.data) < 0:
        raise RuntimeError("theta resampling did not meet the gap floor")
    return t


def dense_normal(n: int, seed: int, tag: str = "delta", symmetric: bool = False) -> np.ndarray:
    a = np.empty((n, n))
    N.problems_lib().dpt_gen_dense_normal(n, seed, tag.encode(), 1 if symmetric else 0, a.ctypes.data)
    return a


def csr_sym_bernoulli(n: int, seed: int, density: float) -> CsrMatrix:
    L = N.problems_lib()
    rp = np.empty(n + 1, dtype=np.int64)
    nnz = L.dpt_gen_csr_sym_bernoulli(n, seed, density, rp.ctypes.data, None, None)
    cols = np.empty(nnz, dtype=np.int32)
    vals = np.empty(nnz)
    L.dpt_gen_csr_sym_bernoulli(n, seed, density, rp.ctypes.data, cols.ctypes.data, vals.ctypes.data)
    return CsrMatrix(n, rp, cols, vals)


def csr_fixed_per_row(n: int, seed: int, per_row: int) -> CsrMatrix:
    rp = np.empty(n + 1, dtype=np.int64)
    cols = np.empty(n * per_row, dtype=np.int32)
    vals = np.empty(n * per_row)
    N.problems_lib().dpt_gen_csr_fixed_per_row(n, seed, per_row, rp.ctypes.data, cols.ctypes.data,
                                               vals.ctypes.data)
    return CsrMatrix(n, rp, cols, vals)


def random_uniform(n: int, seed: int):
    """The reference's build_random_uniform fixture (partition.cpp:133-142)."""
    t = np.empty(n)
    a = np.empty((n, n))
    N.problems_lib().dpt_gen_random_uniform(n, seed, t.ctypes.data, a.ctypes.data)
    return t, a


def oscillator(n: int):
    """The reference's build_oscillator fixture (partition.cpp:98-111)."""
    t = np.empty(n)
    a = np.empty((n, n))
    N.problems_lib().dpt_gen_oscillator(n, t.ctypes.data, a.ctypes.data)
    return t, a


def two_by_two(lam: float) -> PartitionedProblem:  # partition.cpp:98-104 fixture
    return PartitionedProblem(np.array([0.0, 1.0]), np.array([[0.0, 1.0], [1.0, 0.0]]), lam)


def three_by_three(lam: float) -> PartitionedProblem:
    return PartitionedProblem(np.array([0.0, 1.0, 3.0]),
                              np.array([[0.0, 1.0, 2.0], [1.0, 0.0, 3.0], [2.0, 3.0, 0.0]]), lam)


# ---- BASELINE.json configs; n can be scaled down for tests ----
def config(name: str, n: int = None) -> tuple:
    """Returns (PartitionedProblem, IterationOptions kwargs, description)."""
    if name == "c1":  # dense symmetric, seed 0, theta_i = i, lambda 0.05
        n = n or 1024
        return (PartitionedProblem(theta_linear(n), dense_normal(n, 0, "delta", True), 0.05),
                dict(tol=1e-12, max_iter=1000), f"dense symmetric n={n} seed 0 lambda 0.05")
    if name in ("c2", "c2b"):  # dense unsymmetric, seed 1, lambda 0.5/sqrt(n)
        n = n or 4096
        th = theta_uniform_sorted(n, 1, float(n), 1e-3) if name == "c2" else theta_linear(n)
        return (PartitionedProblem(th, dense_normal(n, 1, "delta", False), 0.5 / math.sqrt(n)),
                dict(tol=1e-12, max_iter=500), f"dense unsymmetric n={n} seed 1 lambda 0.5/sqrt(n)"
                + (" (companion 2b: theta_i = i)" if name == "c2b" else ""))
    if name == "c3":  # CSR symmetric 0.5%, seed 2, theta_i = i, lambda 0.1
        n = n or 8192
        return (PartitionedProblem(theta_linear(n), csr_sym_bernoulli(n, 2, 0.005), 0.1),
                dict(tol=1e-12), f"CSR symmetric n={n} density 0.5% seed 2 lambda 0.1")
    if name in ("c4", "c4b"):  # single vector, 16 nnz/row, seed 3, theta_i = i/n (4i/n for 4b)
        n = n or (1 << 20)
        scale = (1.0 if name == "c4" else 4.0) / n
        return (PartitionedProblem(theta_linear(n, scale), csr_fixed_per_row(n, 3, 16), 0.01),
                dict(tol=1e-12), f"CSR 16/row n={n} seed 3 lambda 0.01 theta_i={'4' if name == 'c4b' else ''}i/n")
    if name == "c5":  # dense symmetric, seed 4, lambda 0.5/sqrt(n)
        n = n or 32768
        return (PartitionedProblem(theta_linear(n), dense_normal(n, 4, "delta", True), 0.5 / math.sqrt(n)),
                dict(tol=1e-12), f"dense symmetric n={n} seed 4 lambda 0.5/sqrt(n)")
    raise KeyError(name)
