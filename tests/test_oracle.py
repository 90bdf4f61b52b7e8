"""CPU: pin the oracle (the C restatement) -- bit-exact against the reference
library itself (oracle/_ref) and against the committed golden fixtures that the
reference produced (tests/golden/make_golden.py), plus the reference's own
known-answer tests for this path (proj/tests/test_dpt.cpp, test_partition.cpp)
restated for real inputs."""
import math

import numpy as np
import pytest

from oracle.bind import Checker, available
from paper_2002_12872_b200 import problems as pr
from paper_2002_12872_b200.dpt import PartitionedProblem

from helpers import dominant_fixtures, full_fixtures, load_dominant, load_full

O = Checker("oracle")
REF = pytest.mark.skipif(not available("reference"), reason="oracle/_ref not built (no /root/reference here)")


def same(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b), equal_nan=True)


# ------------------------------------------------------------ golden pins ----
@pytest.mark.parametrize("path", full_fixtures(), ids=lambda p: p.split("/")[-1])
def test_restatement_matches_reference_golden_full(path):
    p, opts, z = load_full(path)
    r = O.iterate_full(p, opts, trace=True)
    assert r.status == int(z["status"]) and r.iterations == int(z["iterations"])
    assert r.step_norm == float(z["step_norm"])
    assert same(r.a, z["a"]) and same(r.eig, z["eig"]) and same(r.res, z["res"])
    assert same(r.trace_step, z["trace_step"]) and same(r.trace_res, z["trace_res"])
    rc, a2 = O.iterate_fixed(p, 2, p.lam)
    assert rc == 0 and same(a2, z["fixed2"])


@pytest.mark.parametrize("path", dominant_fixtures(), ids=lambda p: p.split("/")[-1])
def test_restatement_matches_reference_golden_dominant(path):
    p, z = load_dominant(path)
    r = O.dominant_eigenpair(p, {})
    assert r.status == int(z["status"]) and r.iterations == int(z["iterations"]) and r.row == int(z["row"])
    assert r.eigenvalue == float(z["eigenvalue"]) and r.residual == float(z["residual"])
    assert same(r.z, z["z"]) and same(r.z_unit, z["z_unit"])


# ----------------------------------------------- live reference bit-exactness ----
@REF
@pytest.mark.parametrize("name,n", [("c1", 33), ("c2", 40), ("c2b", 57), ("c3", 130)])
def test_restatement_bit_exact_vs_reference(name, n):
    R = Checker("reference")
    p, o, _ = pr.config(name, n)
    for ramped, alpha in [(False, 0.0), (True, 0.5)]:
        a = O.iterate_full(p, o, trace=True, ramped=ramped, alpha=alpha)
        b = R.iterate_full(p, o, trace=True, ramped=ramped, alpha=alpha)
        assert (a.status, a.iterations, a.step_norm) == (b.status, b.iterations, b.step_norm)
        assert same(a.a, b.a) and same(a.eig, b.eig) and same(a.res, b.res)
        assert same(a.trace_step, b.trace_step) and same(a.trace_res, b.trace_res)
        assert b.imag_max == 0.0  # real inputs keep exactly-zero imaginary parts
    z = np.random.default_rng(5).standard_normal(n)
    assert same(O.step_single(z, 3, p, 0.07), R.step_single(z, 3, p, 0.07))
    assert O.eigenvalue_of(z, 3, p, 0.07) == R.eigenvalue_of(z, 3, p, 0.07)
    A = np.random.default_rng(6).standard_normal((n, n))
    assert same(O.step_full(A, p, 0.07), R.step_full(A, p, 0.07))
    assert same(O.step_rows(p, 5, A[5:9], 0.07), R.step_rows(p, 5, A[5:9], 0.07))
    assert same(O.step_rows(p, 5, A[5:9], 0.07), O.step_full(A, p, 0.07)[5:9])


@REF
@pytest.mark.parametrize("n,per_row,seed", [(300, 4, 1), (512, 16, 3)])
def test_row_map_bit_exact_vs_reference(n, per_row, seed):
    R = Checker("reference")
    csr = pr.csr_fixed_per_row(n, seed, per_row)
    for scale in (4.0 / n, 1.0 / n):
        p = PartitionedProblem(pr.theta_linear(n, scale), csr, 0.01)
        a, b = O.dominant_eigenpair(p, {}), R.dominant_eigenpair(p, {})
        assert (a.status, a.iterations, a.row, a.eigenvalue, a.residual) == \
               (b.status, b.iterations, b.row, b.eigenvalue, b.residual)
        assert same(a.z, b.z) and same(a.z_unit, b.z_unit)
        for ramp in (0.0, 0.3):
            a = O.iterate_single(p, 7, {"max_iter": 60}, ramp, trace=True)
            b = R.iterate_single(p, 7, {"max_iter": 60}, ramp, trace=True)
            assert (a.status, a.iterations, a.eigenvalue, a.residual) == (b.status, b.iterations, b.eigenvalue, b.residual)
            assert same(a.z, b.z) and same(a.trace_step, b.trace_step) and same(a.trace_res, b.trace_res)


@REF
def test_degeneracy_payload_matches_reference():
    R = Checker("reference")
    rng = np.random.default_rng(0)
    for trial in range(40):
        n = int(rng.integers(2, 30))
        d = rng.integers(0, n, size=n).astype(float) * 0.5
        if trial % 3 == 0:
            d = np.sort(d)
        assert O.check_degenerate(d) == R.check_degenerate(d)
    d = np.array([0.0, 1e-16, 2.0])  # test_partition.cpp:97-109
    assert R.check_degenerate(d) == (0, 1) == O.check_degenerate(d)


# ---------------------------------------- known answers (test_dpt.cpp) ----
def test_first_step_from_identity():  # test_dpt.cpp:34-43
    a1 = O.step_full(np.eye(2), pr.two_by_two(0.3), 0.3)
    assert a1[0, 0] == 1.0 and a1[1, 1] == 1.0
    assert abs(a1[0, 1] + 0.3) < 1e-16 and abs(a1[1, 0] - 0.3) < 1e-16


def test_unit_diagonal_exact():  # test_dpt.cpp:45-53 (real lambda)
    t, d = pr.random_uniform(5, 17)
    p = PartitionedProblem(t, d, 0.05)
    a = np.eye(5)
    for _ in range(50):
        a = O.step_full(a, p, 0.05)
        assert np.all(np.diag(a) == 1.0)


def test_two_level_fixed_point():  # test_dpt.cpp:74-90
    r = O.iterate_full(pr.two_by_two(0.3), {})
    assert r.status == 0 and r.iterations > 1 and r.step_norm < 1e-12
    s = math.sqrt(1 + 4 * 0.09)
    assert abs(r.eig[0] - (1 - s) / 2) < 1e-12 and abs(r.eig[1] - (1 + s) / 2) < 1e-12
    xs = (1 - s) / 0.6
    assert abs(r.a[0, 1] - xs) < 1e-12 and abs(r.a[1, 0] + xs) < 1e-12
    assert np.all(r.res < 1e-10)


def test_zero_coupling_and_divergence_and_cycle():  # test_dpt.cpp:92-121
    r = O.iterate_full(pr.two_by_two(0.0), {})
    assert (r.status, r.iterations) == (0, 1) and r.eig[0] == 0.0 and r.eig[1] == 1.0
    r = O.iterate_full(pr.two_by_two(2.0), {})
    assert r.status == 2 and r.iterations < 10000 and np.all(np.isnan(r.eig))
    r = O.iterate_full(pr.two_by_two(0.88), {})
    assert r.status == 1
    r = O.iterate_full(pr.two_by_two(0.88), {"cycle_window": 0, "max_iter": 500})
    assert (r.status, r.iterations) == (3, 500)


def test_budget_and_residual_gate_and_trace():  # test_dpt.cpp:123-156
    r = O.iterate_full(pr.two_by_two(0.3), {"max_iter": 3})
    assert (r.status, r.iterations) == (3, 3) and np.all(np.isfinite(r.a)) and np.all(np.isfinite(r.eig))
    r = O.iterate_full(pr.two_by_two(0.3), {"residual_tol": 0.0, "max_iter": 300})
    assert r.status == 3 and r.step_norm < 1e-12
    r = O.iterate_full(pr.two_by_two(0.3), {}, trace=True)
    assert len(r.trace_step) == r.iterations and r.trace_res[-1] < 1e-10 and r.trace_step[-1] < 1e-12


def test_fixed_and_ramped():  # test_dpt.cpp:167-199
    p = pr.two_by_two(0.21)
    assert abs(O.iterate_fixed(p, 1, 0.21)[1][0, 1] + 0.21) < 1e-16
    want = 0.21 ** 3 - 0.21
    a2 = O.iterate_fixed(p, 2, 0.21)[1]
    assert abs(a2[0, 1] - want) < 1e-15 and abs(a2[1, 0] + want) < 1e-15
    p = pr.two_by_two(0.3)
    plain = O.iterate_full(p, {})
    ramp0 = O.iterate_full(p, {}, ramped=True, alpha=0.0)
    assert ramp0.iterations == plain.iterations + 1
    assert np.max(np.abs(ramp0.eig - plain.eig)) < 1e-14
    ramp7 = O.iterate_full(p, {}, ramped=True, alpha=0.7)
    assert ramp7.status == 0 and np.max(np.abs(ramp7.a - plain.a)) < 1e-10 and ramp7.iterations > plain.iterations


def test_single_row_known_answers():  # test_dpt.cpp:158-233
    p = pr.two_by_two(0.3)
    s = math.sqrt(1 + 4 * 0.09)
    assert abs(O.eigenvalue_of(np.array([1.0, (1 - s) / 0.6]), 0, p, 0.3) - (1 - s) / 2) < 1e-14
    r = O.iterate_single(p, 0)
    assert r.status == 0 and r.z[0] == 1.0 and abs(r.z[1] - (1 - s) / 0.6) < 1e-12 and r.residual < 1e-10
    assert O.iterate_single(pr.two_by_two(2.0), 0).status == 2
    assert O.iterate_single(pr.two_by_two(0.88), 0).status == 1
    t, d = pr.random_uniform(5, 31)
    p = PartitionedProblem(t, d, 0.03)
    full = O.iterate_full(p, {})
    assert full.status == 0
    for row in range(5):
        r = O.iterate_single(p, row)
        assert r.status == 0 and abs(r.eigenvalue - full.eig[row]) < 1e-10
        assert np.max(np.abs(r.z - full.a[row])) < 1e-9


def test_dominant_known_answers():  # test_dpt.cpp:235-276
    p = PartitionedProblem(np.array([0.0, 1.0, 3.0]), np.zeros((3, 3)), 1.0)
    r = O.dominant_eigenpair(p, {})
    assert (r.status, r.row, r.iterations) == (0, 2, 1) and r.eigenvalue == 3.0
    assert abs(np.linalg.norm(r.z_unit) - 1) < 1e-14
    p = PartitionedProblem(np.array([0.0, 2.0, 2.0 + 1e-15]), np.zeros((3, 3)), 1.0)
    assert O.dominant_eigenpair(p, {}).rc == 2
    t, d = pr.oscillator(40)
    p = PartitionedProblem(t, d, 0.5)
    r = O.dominant_eigenpair(p, {})
    assert r.status == 0 and r.row == 39 and r.residual < 1e-10
    w = np.linalg.eigvalsh(np.diag(t) + 0.5 * d)
    assert abs(r.eigenvalue - w[-1]) < 1e-8


def test_effective_window():  # dpt.cpp:83-90
    import ctypes
    L = O.L
    assert L.orc_effective_window(16, 1024) == 3
    assert L.orc_effective_window(16, 1415) == 0
    assert L.orc_effective_window(16, 100) == 16
    assert L.orc_effective_window(1, 10) == 0
    assert L.orc_effective_window(0, 10) == 0


@pytest.mark.parametrize("name,n", [("c2", 300), ("c5", 700)])
def test_gen_matches_inputs(name, n):
    """oracle/gen.py (the reference arm's input builder, numpy) restates the
    §8(d) recipe: the integer stream is bit-identical to csrc/problems.cpp, so
    theta is identical and Delta agrees to the last ulp of numpy's log/cos."""
    from oracle import gen
    from paper_2002_12872_b200 import problems as pr
    t, a, lam = gen.dense_config(name, n)
    p, _, _ = pr.config(name, n)
    assert np.array_equal(t, p.d) and lam == p.lam
    assert np.max(np.abs(a - p.delta)) <= 4 * np.finfo(float).eps * max(1.0, np.max(np.abs(p.delta)))
    assert np.array_equal(a == 0, p.delta == 0)
    if name == "c5":
        assert np.array_equal(a, a.T)
