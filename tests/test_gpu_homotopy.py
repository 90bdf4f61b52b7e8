"""GPU: staged continuation homotopy_solve on the device (SURVEY.md §8(f) row
f2) against the reference's homotopy_solve (proj/src/dpt.cpp:505-556, in
oracle/_ref).  The basis algebra runs in the library-free DMMA GEMM + cluster LU (csrc/linalg.cu) and each stage in
the solver's kernels, so parity is numerical: same status, iterations within
+-1 per stage, eigenvalues 1e-10 relative, eigenvectors 1e-9 max-abs.  Plus
the reference's own homotopy tests (proj/tests/test_dpt.cpp:336-359)."""
import numpy as np
import pytest

import paper_2002_12872_b200 as P
from oracle.bind import ComplexReference, available
from paper_2002_12872_b200 import problems as pr
from paper_2002_12872_b200.dpt import IterationOptions, PartitionedProblem

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not available("reference"), reason="oracle/_ref not built")]

EIG_RTOL, VEC_ATOL = 1e-10, 1e-9


@pytest.fixture(scope="module")
def R():
    return ComplexReference()


def two_level(lam):
    s = np.sqrt(1 + 4 * lam * lam + 0j)
    return (1 - s) / 2, (1 + s) / 2


def compare(R, p, stages, opts=None):
    """Both implementations on p: the same error, or the same report."""
    r = R.homotopy(p, stages, opts or {})
    if r.rc == 2:  # DegenerateSpectrum in some stage (or the base problem)
        with pytest.raises(P.DegenerateSpectrum):
            P.homotopy_solve(p, stages, IterationOptions(**(opts or {})))
        return None
    assert r.rc == 0
    g = P.homotopy_solve(p, stages, IterationOptions(**(opts or {})))
    check(g, r, stages)
    return g


def check(g, r, stages):
    assert int(g.status) == r.status
    assert abs(g.iterations - r.iterations) <= stages, (g.iterations, r.iterations)
    if r.status != 2:
        rel = np.max(np.abs(g.eigenvalues - r.eig) / np.maximum(1.0, np.abs(r.eig)))
        assert rel < EIG_RTOL, rel
        assert np.max(np.abs(g.state.a - r.a)) < VEC_ATOL


def test_reference_known_answers():
    p = pr.two_by_two(1.2)
    assert P.iterate_full(p).status != P.ConvergenceStatus.Converged
    h = P.homotopy_solve(p, 4)
    assert h.status == P.ConvergenceStatus.Converged
    lo, hi = two_level(1.2)
    assert abs(h.eigenvalues[0] - lo) < 1e-9 and abs(h.eigenvalues[1] - hi) < 1e-9
    assert np.all(h.residuals < 1e-9)
    with pytest.raises(ValueError):
        P.homotopy_solve(p, 0)
    p = pr.two_by_two(0.3)
    d, h = P.iterate_full(p), P.homotopy_solve(p, 1)
    assert h.status == P.ConvergenceStatus.Converged
    assert np.max(np.abs(h.eigenvalues - d.eigenvalues)) < 1e-12
    assert np.max(np.abs(h.state.a - d.state.a)) < 1e-10


@pytest.mark.parametrize("n,seed,lam,stages", [(6, 3, 0.2, 3), (7, 4, 0.2, 2), (16, 5, 0.1, 4), (33, 6, 0.08, 2),
                                               (40, 1, 0.05, 2), (40, 2, 0.05, 2), (130, 2, 0.02, 3),
                                               (161, 3, 0.02, 2)])
def test_random_uniform_vs_reference(R, n, seed, lam, stages):
    t, d = pr.random_uniform(n, seed)
    compare(R, PartitionedProblem(t, d, lam), stages)


def test_oscillator_vs_reference(R):
    t, d = pr.oscillator(48)
    g = compare(R, PartitionedProblem(t, d, 0.3), 3)
    assert g is not None and g.status == P.ConvergenceStatus.Converged


def test_complex_coupling_and_levels(R):
    rng = np.random.default_rng(2)
    n = 24
    d = np.arange(n, dtype=float) + 1j * rng.uniform(-0.2, 0.2, n)
    D = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
    compare(R, PartitionedProblem(d, D, 0.03 + 0.02j), 3)
    t, dd = pr.random_uniform(8, 4)
    compare(R, PartitionedProblem(t, dd, 0.15 + 0.1j), 2)


def test_csr_delta_and_stalled_stage(R):
    c = pr.csr_sym_bernoulli(200, 7, 0.05)
    compare(R, PartitionedProblem(np.arange(200, dtype=float), c, 0.08), 2)
    # a stage that does not converge ends the continuation with its status
    p = pr.two_by_two(2.0)
    g, r = P.homotopy_solve(p, 1, IterationOptions(max_iter=50)), R.homotopy(p, 1, {"max_iter": 50})
    assert int(g.status) == r.status and g.iterations == r.iterations


def test_c1_scale(R):
    """n = 1024 (c1), 2 stages: the stage solves are K1 launches, the basis algebra csrc/linalg.cu."""
    p, o, _ = pr.config("c1", 1024)
    g = P.homotopy_solve(p, 2, IterationOptions(**o))
    assert g.status == P.ConvergenceStatus.Converged
    assert np.max(g.residuals) < 1e-9
    # the final eigenvalues agree with the direct solve's (same fixed point)
    direct = P.iterate_full(p, IterationOptions(**o))
    assert np.max(np.abs(np.sort(g.eigenvalues.real) - np.sort(direct.eigenvalues.real))) < 1e-9
