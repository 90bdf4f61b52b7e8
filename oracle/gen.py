"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the SURVEY.md §8(d) input
recipe (the reference's Rng, proj/include/dynspec/rng.hpp:12-54: splitmix64,
streams seed XOR FNV-1a(tag), uniform01 = (u64 >> 11) 2^-53; Box-Muller cos
branch) for the dense configs, so that bench.py's reference arm builds its
inputs without loading any of the product's shared libraries.

splitmix64's k-th output only depends on state0 + (k+1) * gamma, so a whole
n x n matrix is drawn vectorised.  The integer stream is bit-identical to
paper_2002_12872_b200/csrc/problems.cpp; log / cos come from numpy's SIMD
ufuncs, which may differ from glibc's in the last ulp -- same distribution,
values equal to ~1e-15 relative (tests/test_oracle.py::test_gen_matches_inputs).
"""
from __future__ import annotations

import math

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def fnv1a(tag: str) -> int:
    h = 1469598103934665603
    for c in tag.encode():
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def draws(seed: int, tag: str, start: int, count: int) -> np.ndarray:
    """Outputs start .. start+count-1 of Rng::stream(seed, tag).next()."""
    s0 = np.uint64((seed ^ fnv1a(tag)) & 0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        k = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = s0 + k * GAMMA
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        return z ^ (z >> np.uint64(31))


def uniform01(u: np.ndarray) -> np.ndarray:
    return (u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def dense_normal(n: int, seed: int, tag: str = "delta", symmetric: bool = False, chunk_rows: int = 256):
    """Row-major N(0,1) draws (u1 then u2 per entry), optionally symmetrised as
    (X + X^T)/2, zero diagonal (problems.cpp dpt_gen_dense_normal)."""
    a = np.empty((n, n))
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        u = uniform01(draws(seed, tag, 2 * r0 * n, 2 * (r1 - r0) * n))
        u1, u2 = u[0::2], u[1::2]
        a[r0:r1] = (np.sqrt(-2.0 * np.log(1.0 - u1)) * np.cos(2.0 * math.pi * u2)).reshape(r1 - r0, n)
    if symmetric:  # tile by tile: (x + y) / 2 is symmetric in x, y, so each pair gets one value
        b = 1024
        for i0 in range(0, n, b):
            for j0 in range(i0, n, b):
                v = (a[i0:i0 + b, j0:j0 + b] + a[j0:j0 + b, i0:i0 + b].T) / 2.0
                a[i0:i0 + b, j0:j0 + b] = v
                a[j0:j0 + b, i0:i0 + b] = v.T
    np.fill_diagonal(a, 0.0)
    return a


def theta_uniform_sorted(n: int, seed: int, hi: float, min_gap: float) -> np.ndarray:
    k = 0
    while True:
        t = np.sort(0.0 + (hi - 0.0) * uniform01(draws(seed, "theta", k, n)))
        k += n
        if n < 2 or np.min(np.diff(t)) >= min_gap:
            return t


def dense_config(name: str, n: int = None):
    """(theta, Delta, lambda) of BASELINE configs[1] (c2) and configs[4] (c5)."""
    if name == "c2":
        n = n or 4096
        return theta_uniform_sorted(n, 1, float(n), 1e-3), dense_normal(n, 1, "delta", False), 0.5 / math.sqrt(n)
    if name == "c5":
        n = n or 32768
        return np.arange(n, dtype=np.float64), dense_normal(n, 4, "delta", True), 0.5 / math.sqrt(n)
    raise KeyError(name)
