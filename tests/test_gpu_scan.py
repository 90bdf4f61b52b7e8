"""GPU: batched scan_domain against the reference's
own scan_domain (proj/src/analysis.cpp:68-138, compiled in oracle/_ref).

The batched kernel restates run_full / run_single operation by operation, so
the per-cell classes AND iteration counts must be identical to the
reference's (exact equality, no tolerance).  Problems larger than the batched
limit fall back to one GPU solve per cell; those are checked on classes, with
iterations within +-1 (the solver's GEMM order differs from the reference's)."""
import numpy as np
import pytest

import paper_2002_12872_b200 as P
from oracle.bind import ComplexReference, available
from paper_2002_12872_b200 import problems as pr
from paper_2002_12872_b200.dpt import CsrMatrix, IterationOptions, PartitionedProblem, ScanGrid, ScanMode

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not available("reference"), reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def R():
    return ComplexReference()


def run_both(R, p, grid, mode="Full", row=0, alpha=0.0, opts=None):
    o = IterationOptions(**(opts or {}))
    g = P.scan_domain(p, grid, ScanMode(mode, row, alpha), o)
    rc, cls, its, _ = R.scan_domain(p, grid, mode, row, alpha, opts or {}, threads=16)
    assert rc == 0
    return g, cls, its


def assert_exact(g, cls, its):
    bad = np.argwhere((g.classes != cls) | (g.iterations != its))
    assert bad.size == 0, (bad[:5], g.classes[tuple(bad[0])], cls[tuple(bad[0])], g.iterations[tuple(bad[0])],
                           its[tuple(bad[0])])


@pytest.mark.parametrize("mode,row", [("Full", 0), ("SingleRow", 1)])
def test_two_by_two_lambda_plane(R, mode, row):
    grid = ScanGrid(-1.2, 1.2, -1.0, 1.0, 61, 41)
    g, cls, its = run_both(R, pr.two_by_two(1.0), grid, mode, row, opts={"max_iter": 400})
    assert_exact(g, cls, its)
    # all three classes occur (the plane crosses the contraction boundary)
    assert set(np.unique(g.classes)) == {0, 1, 2}


def test_three_by_three_full_and_rows(R):
    grid = ScanGrid(0.0, 0.9, -0.5, 0.5, 37, 23)
    p = pr.three_by_three(1.0)
    for mode, row in (("Full", 0), ("SingleRow", 0), ("SingleRow", 2)):
        assert_exact(*run_both(R, p, grid, mode, row, opts={"max_iter": 300}))


@pytest.mark.parametrize("n,seed", [(5, 17), (6, 3), (8, 11), (13, 2), (24, 5), (32, 9)])
def test_random_uniform_full(R, n, seed):
    t, d = pr.random_uniform(n, seed)
    grid = ScanGrid(-0.4, 0.4, -0.3, 0.3, 19, 13)
    assert_exact(*run_both(R, PartitionedProblem(t, d, 0.0), grid, "Full", 0, opts={"max_iter": 200}))


def test_ramped_and_window_options(R):
    t, d = pr.random_uniform(6, 4)
    p = PartitionedProblem(t, d, 0.0)
    grid = ScanGrid(-0.5, 0.5, -0.5, 0.5, 17, 17)
    for mode in ("Full", "SingleRow"):
        assert_exact(*run_both(R, p, grid, mode, 3, alpha=0.5, opts={"max_iter": 150}))
        assert_exact(*run_both(R, p, grid, mode, 3, opts={"max_iter": 150, "cycle_window": 0}))
        assert_exact(*run_both(R, p, grid, mode, 3, opts={"max_iter": 150, "cycle_window": 3, "tol": 1e-9}))


def test_complex_levels_and_sparse_delta(R):
    rng = np.random.default_rng(7)
    n = 10
    d = np.arange(n, dtype=float) + 1j * rng.uniform(-0.3, 0.3, n)
    D = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
    D[rng.uniform(size=(n, n)) < 0.5] = 0.0
    grid = ScanGrid(-0.3, 0.3, -0.2, 0.2, 15, 11)
    p = PartitionedProblem(d, D, 0.0)
    assert_exact(*run_both(R, p, grid, "Full", opts={"max_iter": 200}))
    # the same matrix as CSR
    rows, cols = np.nonzero(D)
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    rp = np.cumsum(rp)
    csr = CsrMatrix(n, rp, cols.astype(np.int32), D[rows, cols])
    assert_exact(*run_both(R, PartitionedProblem(d, csr, 0.0), grid, "SingleRow", 4, opts={"max_iter": 200}))


def test_row_mode_large_n_batched(R):
    t, d = pr.oscillator(300)
    grid = ScanGrid(0.0, 0.8, -0.2, 0.2, 9, 5)
    assert_exact(*run_both(R, PartitionedProblem(t, d, 0.0), grid, "SingleRow", 299, opts={"max_iter": 300}))


def test_full_mode_fallback_beyond_batched_limit(R):
    t, d = pr.random_uniform(40, 1)
    grid = ScanGrid(-0.05, 0.05, -0.05, 0.05, 3, 3)
    g, cls, its = run_both(R, PartitionedProblem(t, d, 0.0), grid, "Full", opts={"max_iter": 200})
    assert np.array_equal(g.classes, cls)
    assert np.max(np.abs(g.iterations - its)) <= 1


def test_errors_match_reference(R):
    with pytest.raises(P.ShapeError):
        P.scan_domain(pr.two_by_two(0.1), ScanGrid(res_re=0))
    with pytest.raises(P.ShapeError):
        P.scan_domain(pr.two_by_two(0.1), ScanGrid(), ScanMode("SingleRow", 2))
    deg = PartitionedProblem(np.array([0.0, 1.0, 1.0]), np.zeros((3, 3)), 0.0)
    with pytest.raises(P.DegenerateSpectrum) as e:
        P.scan_domain(deg, ScanGrid(res_re=3, res_im=3))
    rc, _, _, (i, j) = R.scan_domain(deg, ScanGrid(res_re=3, res_im=3))
    assert rc == 2 and (e.value.first(), e.value.second()) == (i, j) == (1, 2)
    # SingleRow only validates its own row (build_gap_row)
    g = P.scan_domain(deg, ScanGrid(res_re=3, res_im=3), ScanMode("SingleRow", 0))
    rc, cls, its, _ = R.scan_domain(deg, ScanGrid(res_re=3, res_im=3), "SingleRow", 0)
    assert rc == 0 and np.array_equal(g.classes, cls) and np.array_equal(g.iterations, its)


def test_tiny_thread_per_cell_paths(R):
    """n <= 3 runs one thread per cell: n = 1, 2 (complex Delta), 3 with ramps and tight windows."""
    grid = ScanGrid(-0.9, 0.9, -0.7, 0.7, 33, 29)
    one = PartitionedProblem(np.array([0.5]), np.array([[0.25]]), 0.0)
    for mode in ("Full", "SingleRow"):
        assert_exact(*run_both(R, one, grid, mode, 0))
    two = PartitionedProblem(np.array([0.0, 1.0 + 0.2j]), np.array([[0.1j, 1.0], [1.0 - 0.5j, 0.0]]), 0.0)
    for mode, row in (("Full", 0), ("SingleRow", 1)):
        assert_exact(*run_both(R, two, grid, mode, row, opts={"max_iter": 500}))
        assert_exact(*run_both(R, two, grid, mode, row, alpha=0.3, opts={"max_iter": 200, "cycle_window": 4}))
    three = pr.three_by_three(1.0)
    for mode, row in (("Full", 0), ("SingleRow", 2)):
        assert_exact(*run_both(R, three, grid, mode, row, opts={"max_iter": 0}))
        assert_exact(*run_both(R, three, grid, mode, row, opts={"max_iter": 1000, "cycle_window": 40}))
