"""GPU: degenerate sizes against the reference (oracle/_ref): empty problems
(n = 0, dense and CSR), one-level problems (n = 1), an empty CSR row set,
dominant_eigenpair of an empty problem (ShapeError), and a CSR matrix with
empty rows.  The reference's outcomes: n = 0 converges at k = 1 with no
eigenvalues; n = 1 converges at k = 1 with eps = d + lambda Delta(0,0)."""
import numpy as np
import pytest

import paper_2002_12872_b200 as P
from oracle.bind import ComplexReference, available
from paper_2002_12872_b200.dpt import CsrMatrix, PartitionedProblem

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not available("reference"), reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def R():
    return ComplexReference()


def empty_csr(n):
    return CsrMatrix(n, np.zeros(n + 1, np.int64), np.zeros(0, np.int32), np.zeros(0))


@pytest.mark.parametrize("delta", [np.zeros((0, 0)), empty_csr(0)], ids=["dense", "csr"])
def test_empty_problem(R, delta):
    p = PartitionedProblem(np.zeros(0), delta, 0.1)
    g, r = P.iterate_full(p), R.iterate_full(p, {})
    assert r.rc == 0 and int(g.status) == r.status and g.iterations == r.iterations
    assert g.eigenvalues.shape == (0,) and g.state.a.shape == (0, 0)
    with pytest.raises(P.ShapeError):
        P.dominant_eigenpair(p)
    assert R.dominant_eigenpair(p, {}).rc == 1  # ShapeError in the reference too


@pytest.mark.parametrize("delta", [np.array([[0.2]]), CsrMatrix(1, np.array([0, 1]), np.array([0], np.int32),
                                                                  np.array([0.2]))], ids=["dense", "csr"])
def test_one_level(R, delta):
    p = PartitionedProblem(np.array([0.5]), delta, 0.1)
    g, r = P.iterate_full(p), R.iterate_full(p, {})
    assert int(g.status) == r.status and g.iterations == r.iterations
    assert abs(g.eigenvalues[0] - r.eig[0]) < 1e-15 and abs(g.eigenvalues[0] - 0.52) < 1e-15
    gs, rs = P.iterate_single(p, 0), R.iterate_single(p, 0, {})
    assert int(gs.status) == rs.status and gs.iterations == rs.iterations
    assert abs(gs.eigenvalue - rs.eigenvalue) < 1e-15
    gd = P.dominant_eigenpair(p)
    assert gd.row == 0 and int(gd.status) == 0


def test_csr_with_empty_rows(R):
    n = 64
    rng = np.random.default_rng(3)
    D = rng.normal(size=(n, n))
    D[rng.uniform(size=(n, n)) < 0.9] = 0.0
    D[5] = 0.0
    D[17] = 0.0
    D[:, 40] = 0.0
    np.fill_diagonal(D, 0.0)
    rows, cols = np.nonzero(D)
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    p = PartitionedProblem(np.arange(n, dtype=float), CsrMatrix(n, np.cumsum(rp), cols.astype(np.int32),
                                                               D[rows, cols]), 0.05)
    g, r = P.iterate_full(p), R.iterate_full(p, {})
    assert int(g.status) == r.status and abs(g.iterations - r.iterations) <= 1
    if g.iterations == r.iterations:
        assert np.max(np.abs(g.state.a - r.a)) < 1e-9
    for row in (5, 17, 40):
        gs, rs = P.iterate_single(p, row), R.iterate_single(p, row, {})
        assert int(gs.status) == rs.status and abs(gs.iterations - rs.iterations) <= 1


def test_empty_problem_other_entry_points(R):
    p = PartitionedProblem(np.zeros(0), np.zeros((0, 0)), 0.1)
    assert P.iterate_fixed(p, 3, 0.1).shape == (0, 0)
    assert P.step_full(np.zeros((0, 0)), p, 0.1).shape == (0, 0)
    g = P.scan_domain(p, P.ScanGrid(-1, 1, -1, 1, 4, 3))
    rc, cls, its, _ = R.scan_domain(p, P.ScanGrid(-1, 1, -1, 1, 4, 3))
    assert rc == 0 and np.array_equal(g.classes, cls) and np.array_equal(g.iterations, its)
    # budget and tolerance corners of the empty solve
    for o in ({"max_iter": 0}, {"tol": 0.0, "max_iter": 7}, {"residual_tol": 0.0, "max_iter": 5}):
        g, r = P.iterate_full(p, P.IterationOptions(**o)), R.iterate_full(p, o)
        assert int(g.status) == r.status and g.iterations == r.iterations, (o, g.status, r.status)
