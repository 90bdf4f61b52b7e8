"""GPU: randomized parity sweep against the reference library (oracle/_ref).

Seeded random problems across the entry points and data kinds -- dense and
CSR Delta, real and complex data, plain / ramped full maps, the row map,
dominant_eigenpair, iterate_fixed and single steps, with random options
(tolerances, budgets, cycle windows) -- each compared with the reference's own
implementation at the parity bar (same status, iterations +-1 where the GPU's
summation order may move a boundary decision by one step, eigenvalues 1e-10
relative, eigenvectors 1e-9).  Couplings are drawn around the contraction
radius so all terminal statuses occur."""
import numpy as np
import pytest

import paper_2002_12872_b200 as P
from oracle.bind import ComplexReference, available
from paper_2002_12872_b200.dpt import CsrMatrix, IterationOptions, PartitionedProblem

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not available("reference"), reason="oracle/_ref not built")]

EIG_RTOL, VEC_ATOL = 1e-10, 1e-9


@pytest.fixture(scope="module")
def R():
    return ComplexReference()


def random_problem(rng, n, kind, cplx):
    d = np.sort(rng.uniform(0, n, n)) + np.arange(n) * 0.5  # well-separated levels
    if cplx:
        d = d + 1j * rng.uniform(-0.3, 0.3, n)
    D = rng.normal(size=(n, n))
    if cplx:
        D = D + 1j * rng.normal(size=(n, n))
    np.fill_diagonal(D, 0.0)
    if kind == "csr":
        D[rng.uniform(size=(n, n)) < 0.7] = 0.0
        rows, cols = np.nonzero(D)
        rp = np.zeros(n + 1, np.int64)
        np.add.at(rp, rows + 1, 1)
        return d, CsrMatrix(n, np.cumsum(rp), cols.astype(np.int32), D[rows, cols])
    return d, D


def random_opts(rng):
    o = {}
    if rng.uniform() < 0.5:
        o["max_iter"] = int(rng.integers(1, 300))
    if rng.uniform() < 0.3:
        o["cycle_window"] = int(rng.choice([0, 2, 3, 8, 16]))
    if rng.uniform() < 0.3:
        o["tol"] = float(10.0 ** rng.uniform(-13, -8))
    return o


def scale_lambda(rng, n, cplx):
    r = float(rng.uniform(0.2, 2.5)) / np.sqrt(n) * 0.5
    return r * np.exp(1j * rng.uniform(0, 2 * np.pi)) if cplx else r * rng.choice([-1.0, 1.0])


def check_full(g, r):
    assert int(g.status) == r.status, (int(g.status), r.status, g.iterations, r.iterations)
    assert abs(g.iterations - r.iterations) <= 1, (g.iterations, r.iterations)
    if r.status != 2 and g.iterations == r.iterations:
        assert np.max(np.abs(g.eigenvalues - r.eig) / np.maximum(1.0, np.abs(r.eig))) < EIG_RTOL
        assert np.max(np.abs(g.state.a - r.a)) < VEC_ATOL


@pytest.mark.parametrize("seed", range(24))
def test_full_map_sweep(R, seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.choice([2, 3, 5, 9, 17, 40, 64, 130, 257]))
    kind = "csr" if seed % 3 == 2 else "dense"
    cplx = seed % 4 == 1
    d, D = random_problem(rng, n, kind, cplx)
    p = PartitionedProblem(d, D, scale_lambda(rng, n, cplx))
    o = random_opts(rng)
    if seed % 5 == 3:
        alpha = float(rng.uniform(0.1, 0.8))
        check_full(P.iterate_ramped(p, alpha, IterationOptions(**o)), R.iterate_full(p, o, ramped=True, alpha=alpha))
    else:
        check_full(P.iterate_full(p, IterationOptions(**o)), R.iterate_full(p, o))


@pytest.mark.parametrize("seed", range(16))
def test_row_map_sweep(R, seed):
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.choice([3, 8, 33, 100, 700]))
    kind = "csr" if seed % 2 else "dense"
    cplx = seed % 4 == 3
    d, D = random_problem(rng, n, kind, cplx)
    p = PartitionedProblem(d, D, scale_lambda(rng, n, cplx))
    o = random_opts(rng)
    row = int(rng.integers(0, n))
    alpha = float(rng.uniform(0.1, 0.7)) if seed % 5 == 0 else 0.0
    g = P.iterate_single(p, row, IterationOptions(**o), alpha)
    r = R.iterate_single(p, row, o, alpha)
    assert int(g.status) == r.status and abs(g.iterations - r.iterations) <= 1, (g.status, r.status)
    if r.status != 2 and g.iterations == r.iterations:
        assert np.max(np.abs(g.z - r.z)) < VEC_ATOL
        assert abs(g.eigenvalue - r.eigenvalue) <= EIG_RTOL * max(1.0, abs(r.eigenvalue))
    gd, rd = P.dominant_eigenpair(p, IterationOptions(**o)), R.dominant_eigenpair(p, o)
    assert gd.row == rd.row and int(gd.status) == rd.status and abs(gd.iterations - rd.iterations) <= 1


@pytest.mark.parametrize("seed", range(10))
def test_single_steps_sweep(R, seed):
    rng = np.random.default_rng(3000 + seed)
    n = int(rng.choice([2, 7, 31, 96]))
    cplx = seed % 2 == 1
    d, D = random_problem(rng, n, "dense" if seed % 3 else "csr", cplx)
    lam = scale_lambda(rng, n, cplx)
    p = PartitionedProblem(d, D, lam)
    a = rng.normal(size=(n, n)) + (1j * rng.normal(size=(n, n)) if cplx else 0)
    assert np.max(np.abs(P.step_full(a, p, lam) - R.step_full(a, p, lam))) < 1e-11
    k = int(rng.integers(1, 6))
    assert np.max(np.abs(P.iterate_fixed(p, k, lam) - R.iterate_fixed(p, k, lam))) < 1e-11
    z = rng.normal(size=n) + (1j * rng.normal(size=n) if cplx else 0)
    row = int(rng.integers(0, n))
    want_z, want_e = R.step_single(z, row, p, lam)
    assert np.max(np.abs(P.step_single(z, row, p, lam) - want_z)) < 1e-11
    assert abs(P.eigenvalue_of(z, row, p, lam) - want_e) < 1e-10 * max(1.0, abs(want_e))
