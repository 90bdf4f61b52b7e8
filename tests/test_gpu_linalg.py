"""GPU: the library-free dense linear algebra of the device homotopy
(csrc/linalg.cu) -- the TMA + DMMA GEMM (K1's tile machinery, plain epilogue)
and the LU with partial pivoting (8-CTA cluster panels over distributed
shared memory, GEMM trailing updates, blocked triangular solves) -- against
the REFERENCE's own matmul (proj/src/matrix.cpp:130-143) and
solve_linear_multi (matrix.cpp:468-533) in oracle/_ref, real and complex,
odd and tiny sizes, non-square right-hand sides, panel / block boundaries,
and the singular-matrix error.  Floating point: products within 1e-13
relative to the operands' scale, solves within 1e-10 relative (cond < 1e4)."""
import numpy as np
import pytest

import paper_2002_12872_b200 as P
from oracle.bind import ComplexReference, available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not available("reference"), reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def R():
    return ComplexReference()


def rand(rng, shape, cplx):
    x = rng.standard_normal(shape)
    return x + 1j * rng.standard_normal(shape) if cplx else x


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("m,k,n", [(1, 1, 1), (3, 5, 7), (17, 33, 9), (64, 64, 64), (127, 129, 131), (300, 16, 513),
                                   (1000, 700, 333)])
def test_matmul_vs_reference(R, m, k, n, cplx):
    rng = np.random.default_rng(m * 7 + k * 3 + n)
    a, b = rand(rng, (m, k), cplx), rand(rng, (k, n), cplx)
    got = P.matmul_dense(a, b)
    want = R.matmul(a, b)
    scale = np.sqrt(k) * 4
    assert np.max(np.abs(got - want)) < 1e-13 * scale * 8
    if not cplx:
        assert got.dtype == np.float64


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("n,nrhs", [(1, 1), (2, 3), (5, 5), (31, 2), (32, 32), (33, 40), (65, 65), (129, 7),
                                    (300, 300), (517, 100), (1024, 64)])
def test_solve_linear_multi_vs_reference(R, n, nrhs, cplx):
    rng = np.random.default_rng(n * 31 + nrhs)
    a = rand(rng, (n, n), cplx) + 4 * np.sqrt(n) * np.eye(n) * rng.choice([-1, 1], n)  # well conditioned
    b = rand(rng, (n, nrhs), cplx)
    got = P.solve_linear_multi(a, b)
    rc, want = R.solve_linear_multi(a, b)
    assert rc == 0
    assert np.max(np.abs(got - want)) <= 1e-10 * max(1.0, np.max(np.abs(want)))
    assert np.max(np.abs(a @ got - b)) <= 1e-10 * np.max(np.abs(b)) * n


@pytest.mark.parametrize("cplx", [False, True])
def test_solve_needs_pivoting(R, cplx):
    """Zero diagonal everywhere (no LU without row interchanges), and a
    permutation matrix: the pivot rule (first row of maximal |a(i,k)|)
    decides every step."""
    rng = np.random.default_rng(3)
    n = 200
    a = rand(rng, (n, n), cplx)
    np.fill_diagonal(a, 0.0)
    b = rand(rng, (n, 5), cplx)
    got = P.solve_linear_multi(a, b)
    rc, want = R.solve_linear_multi(a, b)
    assert rc == 0
    assert np.max(np.abs(a @ got - b)) <= 1e-9 * np.max(np.abs(b)) * n
    assert np.max(np.abs(got - want)) <= 1e-8 * max(1.0, np.max(np.abs(want)))
    perm = rng.permutation(97)
    pm = np.eye(97)[perm] * (1 + 1j if cplx else 1)
    rhs = rand(rng, (97, 3), cplx)
    assert np.max(np.abs(P.solve_linear_multi(pm, rhs) - R.solve_linear_multi(pm, rhs)[1])) < 1e-15


@pytest.mark.parametrize("cplx", [False, True])
def test_singular_matrix_raises(R, cplx):
    rng = np.random.default_rng(5)
    a = rand(rng, (70, 70), cplx)
    a[:, 40] = 0.0  # an exactly-zero column: the reference's "solve_linear: singular matrix"
    b = rand(rng, (70, 2), cplx)
    assert R.solve_linear_multi(a, b)[0] == 8
    with pytest.raises(RuntimeError, match="singular"):
        P.solve_linear_multi(a, b)
    z = np.zeros((3, 3), dtype=np.complex128 if cplx else np.float64)
    with pytest.raises(RuntimeError, match="singular"):
        P.solve_linear_multi(z, np.ones((3, 1)))


def test_large_solve_residual():
    """n = 4096 (the c2b homotopy's size): 128 panels of 32 columns on the
    cluster, residual of the n right-hand-side solve."""
    rng = np.random.default_rng(11)
    n = 4096
    a = rng.standard_normal((n, n)) + 3 * np.sqrt(n) * np.eye(n)
    b = rng.standard_normal((n, 64))
    x = P.solve_linear_multi(a, b)
    assert np.max(np.abs(a @ x - b)) <= 1e-10 * np.max(np.abs(b)) * np.sqrt(n)
    assert np.max(np.abs(x - np.linalg.solve(a, b))) <= 1e-11


def test_empty_and_degenerate_shapes(R):
    """n = 0 / k = 0 / nrhs = 0 (the reference returns empty or zero
    matrices) and 1 x 1 systems."""
    assert P.matmul_dense(np.zeros((0, 3)), np.zeros((3, 4))).shape == (0, 4)
    z = P.matmul_dense(np.zeros((3, 0)), np.zeros((0, 5)))
    assert z.shape == (3, 5) and np.all(z == 0.0)
    assert P.solve_linear_multi(np.zeros((0, 0)), np.zeros((0, 2))).shape == (0, 2)
    assert P.solve_linear_multi(np.eye(4), np.zeros((4, 0))).shape == (4, 0)
    x = P.solve_linear_multi(np.array([[4.0]]), np.array([[2.0, -8.0]]))
    assert np.array_equal(x, np.array([[0.5, -2.0]]))
    with pytest.raises(ValueError):
        P.solve_linear_multi(np.eye(3), np.ones((4, 1)))
