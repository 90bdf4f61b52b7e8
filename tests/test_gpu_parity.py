"""GPU parity: the CUDA path (through the C ABI, libdpt_b200.so) against the
oracle -- the C restatement, pinned bit-exact to the reference -- and the
reference-generated golden fixtures.  Bar (BASELINE.json north_star): same
status, iterations within +-1, eigenvalues within 1e-10 relative, eigenvectors
within 1e-9 max-abs (FP64).  Full BASELINE sizes are covered by
size-independent properties: row slices of the map (the rows are independent,
so any row sample of A_k must match the oracle's step on those rows), residual
gates, and the reference's terminal status."""
import math

import numpy as np
import pytest

import paper_2002_12872_b200 as P
from oracle.bind import Checker
from paper_2002_12872_b200 import problems as pr
from paper_2002_12872_b200.dpt import CsrMatrix, IterationOptions, PartitionedProblem

from helpers import (EIG_RTOL, VEC_ATOL, assert_full_parity, dominant_fixtures, eig_rel_err, full_fixtures,
                     load_dominant, load_full)

pytestmark = pytest.mark.gpu
O = Checker("oracle")


def _o(d):
    return IterationOptions(**d)


# ---------------------------------------------------- golden (reference) ----
@pytest.mark.parametrize("path", full_fixtures(), ids=lambda p: p.split("/")[-1])
def test_full_vs_reference_golden(path):
    p, opts, z = load_full(path)
    trace = []
    g = P.iterate_full(p, _o(opts), trace=lambda k, s, r: trace.append((k, s, r)))
    assert_full_parity(g, z["status"], int(z["iterations"]), z["a"], z["eig"], z["res"])
    assert [t[0] for t in trace] == list(range(1, len(trace) + 1))
    if len(trace) == len(z["trace_step"]):
        st = np.array([t[1] for t in trace])
        ok = z["trace_step"] > 1e-6
        assert np.allclose(st[ok], z["trace_step"][ok], rtol=1e-6)
    a2 = P.iterate_fixed(p, 2, p.lam)
    assert np.max(np.abs(a2 - z["fixed2"])) < 1e-12


@pytest.mark.parametrize("path", dominant_fixtures(), ids=lambda p: p.split("/")[-1])
def test_dominant_vs_reference_golden(path):
    p, z = load_dominant(path)
    g = P.dominant_eigenpair(p)
    assert int(g.status) == int(z["status"]) and abs(g.iterations - int(z["iterations"])) <= 1
    assert g.row == int(z["row"])
    assert abs(g.eigenvalue - float(z["eigenvalue"])) <= EIG_RTOL * max(1.0, abs(float(z["eigenvalue"])))
    assert np.max(np.abs(g.z_chart - z["z"])) < VEC_ATOL and np.max(np.abs(g.z_unit - z["z_unit"])) < VEC_ATOL


# ------------------------------------------------ oracle, scaled configs ----
@pytest.mark.parametrize("name,n", [("c1", 64), ("c1", 200), ("c1", 1024), ("c2", 256), ("c2", 1000),
                                    ("c2b", 512), ("c2b", 2048), ("c3", 512), ("c3", 2048), ("c1", 2049),
                                    ("c1", 131), ("c3", 1)])
def test_full_vs_oracle(name, n):
    p, o, _ = pr.config(name, n)
    g = P.iterate_full(p, _o(o))
    r = O.iterate_full(p, o)
    assert_full_parity(g, r.status, r.iterations, r.a, r.eig, r.res)


@pytest.mark.parametrize("n", [5, 7, 64, 130])
def test_nonzero_diagonal_perturbation(n):  # build_random_uniform keeps Delta's diagonal
    t, d = pr.random_uniform(n, 17)
    p = PartitionedProblem(t, d, 0.5 / n)
    g = P.iterate_full(p)
    r = O.iterate_full(p, {})
    assert_full_parity(g, r.status, r.iterations, r.a, r.eig, r.res)
    csr = CsrMatrix(n, *_dense_to_csr(d))
    g2 = P.iterate_full(PartitionedProblem(t, csr, 0.5 / n))
    assert_full_parity(g2, r.status, r.iterations, r.a, r.eig, r.res)


def _dense_to_csr(a):
    n = a.shape[0]
    rp, cols, vals = [0], [], []
    for i in range(n):
        nz = np.nonzero(a[i])[0]
        cols += list(nz)
        vals += list(a[i, nz])
        rp.append(len(cols))
    return np.array(rp, np.int64), np.array(cols, np.int32), np.array(vals)


def test_ramped_and_trace():
    p, o, _ = pr.config("c1", 300)
    for alpha in (0.0, 0.5, 0.9):
        tr = []
        g = P.iterate_ramped(p, alpha, _o(o), trace=lambda k, s, r: tr.append((k, s, r)))
        r = O.iterate_full(p, o, trace=True, ramped=True, alpha=alpha)
        assert_full_parity(g, r.status, r.iterations, r.a, r.eig, r.res)
        assert len(tr) == g.iterations
        st = np.array([x[1] for x in tr])[: len(r.trace_step)]
        big = r.trace_step[: len(st)] > 1e-8
        assert np.allclose(st[big], r.trace_step[: len(st)][big], rtol=1e-8)
    with pytest.raises(ValueError):
        P.iterate_ramped(p, 1.0)
    with pytest.raises(ValueError):
        P.iterate_ramped(p, -0.1)


def test_trace_exception_propagates():
    def sink(k, s, r):
        if k == 3:
            raise KeyError("stop")
    with pytest.raises(KeyError):
        P.iterate_full(pr.two_by_two(0.3), trace=sink)


def test_trace_abort_stops_the_device():
    """A sink that aborts at k = 3 stops the solve within one chunk of launches
    (the reference calls the sink inside its loop, dpt.cpp:153-157): a run
    with max_iter 1000 that never terminates on its own (lambda = 0.88 with
    the cycle window off) issues at most a few chunks, and the sink is never
    called again after it raised."""
    ctx = P.Context(0)
    seen = []

    def sink(k, s, r):
        seen.append(k)
        if k == 3:
            raise KeyError("stop")
    l0 = ctx.launches
    with pytest.raises(KeyError):
        P.iterate_full(pr.two_by_two(0.88), P.IterationOptions(cycle_window=0, max_iter=1000), trace=sink, ctx=ctx)
    assert seen == [1, 2, 3]
    assert ctx.launches - l0 < 3 * (4 + 8 + 8), ctx.launches - l0
    ctx.close()


# ------------------------------------------- known answers (test_dpt.cpp) ----
def test_known_answers_full():
    s = math.sqrt(1 + 4 * 0.09)
    a1 = P.step_full(np.eye(2), pr.two_by_two(0.3), 0.3)
    assert a1[0, 0] == 1.0 and a1[1, 1] == 1.0 and abs(a1[0, 1] + 0.3) < 1e-16 and abs(a1[1, 0] - 0.3) < 1e-16
    r = P.iterate_full(pr.two_by_two(0.3))
    assert r.status == P.ConvergenceStatus.Converged and r.iterations > 1 and r.step_norm < 1e-12
    assert abs(r.eigenvalues[0] - (1 - s) / 2) < 1e-12 and abs(r.eigenvalues[1] - (1 + s) / 2) < 1e-12
    assert abs(r.state.a[0, 1] - (1 - s) / 0.6) < 1e-12 and np.all(r.residuals < 1e-10)
    r = P.iterate_full(pr.two_by_two(0.0))
    assert (int(r.status), r.iterations) == (0, 1) and r.eigenvalues[0] == 0.0 and r.eigenvalues[1] == 1.0
    r = P.iterate_full(pr.two_by_two(2.0))
    assert r.status == P.ConvergenceStatus.Diverged and np.all(np.isnan(r.eigenvalues))
    assert P.iterate_full(pr.two_by_two(0.88)).status == P.ConvergenceStatus.BoundedNonConverged
    r = P.iterate_full(pr.two_by_two(0.88), IterationOptions(cycle_window=0, max_iter=500))
    assert (int(r.status), r.iterations) == (3, 500)
    r = P.iterate_full(pr.two_by_two(0.3), IterationOptions(max_iter=3))
    assert (int(r.status), r.iterations) == (3, 3) and np.all(np.isfinite(r.state.a)) and np.all(np.isfinite(r.eigenvalues))
    r = P.iterate_full(pr.two_by_two(0.3), IterationOptions(residual_tol=0.0, max_iter=300))
    assert int(r.status) == 3 and r.step_norm < 1e-12
    a2 = P.iterate_fixed(pr.two_by_two(0.21), 2, 0.21)
    want = 0.21 ** 3 - 0.21
    assert abs(a2[0, 1] - want) < 1e-15 and abs(a2[1, 0] + want) < 1e-15
    assert np.array_equal(P.iterate_fixed(pr.two_by_two(0.21), 0, 0.21), np.eye(2))
    plain = P.iterate_full(pr.two_by_two(0.3))
    ramp0 = P.iterate_ramped(pr.two_by_two(0.3), 0.0)
    assert ramp0.iterations == plain.iterations + 1
    ramp7 = P.iterate_ramped(pr.two_by_two(0.3), 0.7)
    assert np.max(np.abs(ramp7.state.a - plain.state.a)) < 1e-10 and ramp7.iterations > plain.iterations


def test_unit_diagonal_exact_and_step_full_parity():
    t, d = pr.random_uniform(5, 17)
    p = PartitionedProblem(t, d, 0.05)
    a = np.eye(5)
    for _ in range(50):
        b = P.step_full(a, p, 0.05)
        assert np.all(np.diag(b) == 1.0)
        assert np.max(np.abs(b - O.step_full(a, p, 0.05))) < 1e-13 * max(1, np.max(np.abs(b)))
        a = b
    p, o, _ = pr.config("c2", 300)
    A = np.random.default_rng(1).standard_normal((300, 300)) * 0.1
    assert np.max(np.abs(P.step_full(A, p, 0.03) - O.step_full(A, p, 0.03))) < 1e-12


def test_max_iter_zero_and_degenerate():
    p, o, _ = pr.config("c1", 50)
    for mi in (0, -3):
        g = P.iterate_full(p, IterationOptions(max_iter=mi))
        r = O.iterate_full(p, {"max_iter": mi})
        assert int(g.status) == r.status == 3 and g.iterations == r.iterations == mi
        assert np.array_equal(g.state.a, np.eye(50))
        assert eig_rel_err(g.eigenvalues, r.eig) < EIG_RTOL
    d = np.array([0.0, 1e-16, 2.0])
    with pytest.raises(P.DegenerateSpectrum) as e:
        P.iterate_full(PartitionedProblem(d, np.zeros((3, 3)), 0.1))
    assert (e.value.first(), e.value.second()) == (0, 1)
    with pytest.raises(P.DegenerateSpectrum):
        P.iterate_single(PartitionedProblem(d, np.zeros((3, 3)), 0.1), 0)
    P.iterate_single(PartitionedProblem(d, np.zeros((3, 3)), 0.1), 2)  # only its own gaps matter
    with pytest.raises(P.ShapeError):
        P.iterate_single(PartitionedProblem(d, np.zeros((3, 3)), 0.1), 3)


# ------------------------------------------------------------ row map ----
def test_known_answers_single():
    s = math.sqrt(1 + 4 * 0.09)
    p = pr.two_by_two(0.3)
    assert abs(P.eigenvalue_of(np.array([1.0, (1 - s) / 0.6]), 0, p, 0.3) - (1 - s) / 2) < 1e-14
    r = P.iterate_single(p, 0)
    assert int(r.status) == 0 and r.z[0] == 1.0 and abs(r.z[1] - (1 - s) / 0.6) < 1e-12 and r.residual < 1e-10
    assert P.iterate_single(pr.two_by_two(2.0), 0).status == P.ConvergenceStatus.Diverged
    assert P.iterate_single(pr.two_by_two(0.88), 0).status == P.ConvergenceStatus.BoundedNonConverged
    t, d = pr.random_uniform(5, 31)
    p = PartitionedProblem(t, d, 0.03)
    full = P.iterate_full(p)
    for row in range(5):
        r = P.iterate_single(p, row)
        assert int(r.status) == 0 and abs(r.eigenvalue - full.eigenvalues[row]) < 1e-10
        assert np.max(np.abs(r.z - full.state.a[row])) < 1e-9
    dp = PartitionedProblem(np.array([0.0, 1.0, 3.0]), np.zeros((3, 3)), 1.0)
    r = P.dominant_eigenpair(dp)
    assert (int(r.status), r.row, r.iterations) == (0, 2, 1) and r.eigenvalue == 3.0
    with pytest.raises(P.DegenerateSpectrum):
        P.dominant_eigenpair(PartitionedProblem(np.array([0.0, 2.0, 2.0 + 1e-15]), np.zeros((3, 3)), 1.0))
    t, d = pr.oscillator(40)
    r = P.dominant_eigenpair(PartitionedProblem(t, d, 0.5))
    assert int(r.status) == 0 and r.row == 39 and r.residual < 1e-10
    assert abs(r.eigenvalue - np.linalg.eigvalsh(np.diag(t) + 0.5 * d)[-1]) < 1e-8
    assert abs(np.linalg.norm(r.z_unit) - 1.0) < 1e-12


@pytest.mark.parametrize("n,per_row,scale,ramp", [(2048, 16, 1.0, 0.0), (5000, 7, 4.0, 0.0), (3000, 16, 4.0, 0.4),
                                                  (777, 3, 1.0, 0.0)])
def test_single_csr_vs_oracle(n, per_row, scale, ramp):
    p = PartitionedProblem(pr.theta_linear(n, scale / n), pr.csr_fixed_per_row(n, 3, per_row), 0.01)
    for row in (n - 1, n // 2):
        g = P.iterate_single(p, row, IterationOptions(max_iter=200), ramp_alpha=ramp)
        r = O.iterate_single(p, row, {"max_iter": 200}, ramp)
        assert int(g.status) == r.status and abs(g.iterations - r.iterations) <= 1
        if g.iterations == r.iterations and r.status != 2:
            assert np.max(np.abs(g.z - r.z)) < VEC_ATOL
            assert abs(g.eigenvalue - r.eigenvalue) <= EIG_RTOL * max(1, abs(r.eigenvalue))
    z = np.random.default_rng(2).standard_normal(n)
    assert np.max(np.abs(P.step_single(z, 5, p, 0.02) - O.step_single(z, 5, p, 0.02))) < 1e-13
    assert abs(P.eigenvalue_of(z, 5, p, 0.02) - O.eigenvalue_of(z, 5, p, 0.02)) < 1e-12


def test_single_dense_vs_oracle():
    p, o, _ = pr.config("c1", 300)
    for row in (0, 150, 299):
        g = P.iterate_single(p, row, _o(o))
        r = O.iterate_single(p, row, o)
        assert int(g.status) == r.status and abs(g.iterations - r.iterations) <= 1
        assert np.max(np.abs(g.z - r.z)) < VEC_ATOL


@pytest.mark.parametrize("n", [4097, 4608, 16400])
def test_single_dense_gemv_rows_per_warp_vs_oracle(n):
    # dense row map at the sizes where each warp streams 2 (n >= 4096) or 4
    # (n >= 16384) rows at once; odd n takes the scalar tail column
    d = pr.theta_linear(n, 1.0 / n)
    delta = np.random.default_rng(n).standard_normal((n, n))
    np.fill_diagonal(delta, 0.0)
    p = PartitionedProblem(d, delta, 0.5 / math.sqrt(n))
    o = dict(tol=1e-12, max_iter=60)
    for row in (n - 1, n // 3):
        g = P.iterate_single(p, row, _o(o))
        r = O.iterate_single(p, row, o)
        assert int(g.status) == r.status and abs(g.iterations - r.iterations) <= 1, (row, g.status, r.status)
        if int(r.status) != 2:
            assert np.max(np.abs(g.z - r.z)) < VEC_ATOL
            assert abs(g.eigenvalue - r.eigenvalue) <= EIG_RTOL * max(1.0, abs(r.eigenvalue))


# --------------------------------------------- full BASELINE sizes ----
def _row_sample_check(p, plan_rows, lam, k_rows, a_prev):
    want = O.step_rows(p, 0, a_prev[:k_rows], lam)
    return float(np.max(np.abs(plan_rows[:k_rows] - want)))


def test_c1_full_size_vs_oracle():
    p, o, _ = pr.config("c1")  # n = 1024, the reference's CPU-runnable case
    g = P.iterate_full(p, _o(o))
    r = O.iterate_full(p, o)
    assert_full_parity(g, r.status, r.iterations, r.a, r.eig, r.res)
    assert r.status == 0 and r.iterations == 13  # Converged, 13 iterations


def test_c2_full_size_status_and_row_slices():
    p, o, _ = pr.config("c2")  # n = 4096: the oracle needs ~4 min per full iteration, so check row slices
    g = P.iterate_full(p, _o(o))
    assert g.status == P.ConvergenceStatus.Diverged and g.iterations == 4
    plan = P.Plan(p)
    plan.begin()
    a1 = plan.read()
    plan.steps(1)
    a2 = plan.read()
    a1_ref = O.step_rows(p, 0, np.eye(4096)[:64], p.lam)
    assert np.max(np.abs(a1[:64] - a1_ref)) < 1e-15
    assert _row_sample_check(p, a2, p.lam, 64, a1) < 1e-12
    # the diagonal of each row lies in one tile: check a row block away from 0 too
    rows = slice(3000, 3040)
    want = O.step_rows(p, 3000, a1[rows], p.lam)
    assert np.max(np.abs(a2[rows] - want)) < 1e-12


def test_c3_full_size_vs_reference_golden():
    """BASELINE configs[2] at full size against the REFERENCE's own solve
    (tests/golden/c3full_n8192.npz, written by make_golden.py c3full from
    oracle/_ref): status, iterations, all 8192 eigenvalues (1e-10 relative),
    residuals, and two 64-row blocks of the eigenvector matrix (1e-9)."""
    import os
    from helpers import GOLDEN
    z = np.load(os.path.join(GOLDEN, "c3full_n8192.npz"))
    p, o, _ = pr.config("c3")  # n = 8192 CSR, nnz = 336,376 with the recipe
    assert p.delta.nnz == 336376 == int(z["nnz"])
    assert np.sum(p.delta.vals) == float(z["vals_sum"]) and np.sum(p.delta.cols.astype(np.int64)) == int(z["cols_sum"])
    g = P.iterate_full(p, _o(o))
    assert int(g.status) == int(z["status"]) == 0 and abs(g.iterations - int(z["iterations"])) <= 1
    assert int(z["iterations"]) == 18
    assert eig_rel_err(g.eigenvalues, z["eig"]) < EIG_RTOL
    for key in z.files:
        if key.startswith("a_"):
            a, b = (int(x) for x in key.split("_")[1:])
            assert np.max(np.abs(g.state.a[a:b] - z[key])) < VEC_ATOL, key
    assert np.max(g.residuals) < 1e-10
    assert np.allclose(g.residuals, z["res"], rtol=1e-3, atol=1e-13)
    assert np.all(np.diag(g.state.a) == 1.0)


def test_c2b_full_size_vs_reference_golden():
    """The bench's config family at full size, converging: c2b (BASELINE
    configs[1] with theta_i = i; n = 4096 dense unsymmetric) against the
    REFERENCE's own solve (tests/golden/c2bfull_n4096.npz, make_golden.py
    c2bfull, ~20 min in oracle/_ref): status, iterations, all eigenvalues,
    residuals and two 64-row blocks of the eigenvector matrix."""
    import os
    from helpers import GOLDEN
    z = np.load(os.path.join(GOLDEN, "c2bfull_n4096.npz"))
    p, o, _ = pr.config("c2b")
    assert np.sum(p.delta) == float(z["delta_sum"]) and np.sum(p.delta * p.delta) == float(z["delta_sq"])
    g = P.iterate_full(p, _o(o))
    assert int(g.status) == int(z["status"]) == 0 and abs(g.iterations - int(z["iterations"])) <= 1
    assert eig_rel_err(g.eigenvalues, z["eig"]) < EIG_RTOL
    for key in z.files:
        if key.startswith("a_"):
            a, b = (int(x) for x in key.split("_")[1:])
            assert np.max(np.abs(g.state.a[a:b] - z[key])) < VEC_ATOL, key
    assert np.max(g.residuals) < 1e-10
    assert np.allclose(g.residuals, z["res"], rtol=1e-3, atol=1e-13)


def test_c3_full_size_properties():
    p, o, _ = pr.config("c3")  # n = 8192 CSR, nnz = 336,376 with the recipe
    assert p.delta.nnz == 336376
    g = P.iterate_full(p, _o(o))
    assert g.status == P.ConvergenceStatus.Converged and abs(g.iterations - 18) <= 1
    assert np.max(g.residuals) < 1e-10
    assert np.all(np.diag(g.state.a) == 1.0)
    # one more map application leaves the fixed point within tol (row sample, oracle)
    rows = slice(4000, 4016)
    nxt = O.step_rows(p, 4000, g.state.a[rows], p.lam)
    assert np.max(np.abs(nxt - g.state.a[rows])) < 1e-11


def test_c4_full_size_vs_oracle():
    p, o, _ = pr.config("c4")  # n = 2^20, 16 nnz/row
    g = P.dominant_eigenpair(p, _o(o))
    r = O.dominant_eigenpair(p, o)
    assert int(g.status) == r.status and abs(g.iterations - r.iterations) <= 1
    assert g.row == r.row == (1 << 20) - 1
    if r.status != 2 and g.iterations == r.iterations:
        assert np.max(np.abs(g.z_chart - r.z)) < VEC_ATOL
    p, o, _ = pr.config("c4b")
    g = P.dominant_eigenpair(p, _o(o))
    r = O.dominant_eigenpair(p, o)
    assert int(g.status) == r.status == 0 and abs(g.iterations - r.iterations) <= 1
    assert abs(g.eigenvalue - r.eigenvalue) <= EIG_RTOL * max(1, abs(r.eigenvalue))
    assert np.max(np.abs(g.z_chart - r.z)) < VEC_ATOL and np.max(np.abs(g.z_unit - r.z_unit)) < VEC_ATOL


def _step_rows_threaded(p, row0, a_rows, lam, chunk=4):
    """The oracle's step_rows over row chunks on the host cores (rows of the
    map are independent, dpt.cpp:136-144; ctypes releases the GIL)."""
    import concurrent.futures as cf
    import os
    out = np.empty_like(a_rows)
    starts = list(range(0, a_rows.shape[0], chunk))

    def one(s):
        out[s:s + chunk] = O.step_rows(p, row0 + s, a_rows[s:s + chunk], lam)

    with cf.ThreadPoolExecutor(max_workers=min(len(starts), os.cpu_count() or 1)) as ex:
        list(ex.map(one, starts))
    return out


def test_c5_full_size():
    """BASELINE configs[4]: dense symmetric n = 32768 (the north_star's
    multi-GPU config; the reference cannot run it: >= 103 GB of complex n^2
    buffers).  Size-independent properties against the oracle: two 64-row
    blocks of A_1 and A_2 (rows are independent), the residual gate, the exact
    unit diagonal, a fixed-point row sample of the final iterate, and the same
    solve through the 1-rank NCCL collective path, bit for bit."""
    p, o, _ = pr.config("c5")
    n = 32768
    blocks = (0, 20000)
    plan = P.Plan(p)
    plan.begin()
    full1 = plan.read()
    a1 = {r0: full1[r0:r0 + 64].copy() for r0 in blocks}
    del full1
    plan.steps(1)
    full2 = plan.read()
    a2 = {r0: full2[r0:r0 + 64].copy() for r0 in blocks}
    del full2
    plan.close()
    eye = np.eye(n)
    for r0 in blocks:
        want1 = O.step_rows(p, r0, eye[r0:r0 + 64], p.lam)  # k = 1 from A_0 = I
        assert np.max(np.abs(a1[r0] - want1)) < 1e-15, r0
        want2 = _step_rows_threaded(p, r0, a1[r0], p.lam)  # k = 2: a full dense row product
        assert np.max(np.abs(a2[r0] - want2)) < 1e-12, r0
    del eye
    g = P.iterate_full(p, _o(o))
    assert g.status == P.ConvergenceStatus.Converged and g.iterations <= 12, (g.status, g.iterations)
    assert np.max(g.residuals) < 1e-10
    assert np.all(np.diag(g.state.a) == 1.0)
    assert np.all(np.isfinite(g.eigenvalues))
    # eigenvalues are theta_i + lambda (Delta A)_ii: a row sample from the oracle's own read-off
    for r0 in blocks:
        rows = slice(r0, r0 + 16)
        nxt = _step_rows_threaded(p, r0, g.state.a[rows], p.lam)
        assert np.max(np.abs(nxt - g.state.a[rows])) < 1e-11, r0
    iters, a_g, eig_g = g.iterations, g.state.a, g.eigenvalues
    del g
    ctx = P.Context(0)
    try:
        ctx.set_comm(0, 1, P.Context.nccl_unique_id())
        h = P.iterate_full(p, _o(o), ctx=ctx)
        assert int(h.status) == 0 and h.iterations == iters
        assert np.array_equal(h.eigenvalues, eig_g)
        assert np.array_equal(h.state.a, a_g)
    finally:
        ctx.close()
