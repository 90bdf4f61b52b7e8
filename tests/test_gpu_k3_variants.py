"""GPU: every K3 (16-nonzeros-per-row row map) variant -- block-staged trips
(DPT_U16_VARIANT 0-5) and per-warp pipelines (6-10) -- against the oracle,
and the lane-rotated ones bit for bit against each other (same per-row
accumulation order).  Sizes include a ragged last trip and n smaller than one
warp-trip."""
import os

import numpy as np
import pytest

import paper_2002_12872_b200 as P
from oracle.bind import Checker
from paper_2002_12872_b200 import problems as pr

pytestmark = pytest.mark.gpu

ROTATED = [1, 3, 4, 5, 6, 7, 8, 9, 10, 11, 16, 17, 18, 19, 20]


@pytest.fixture
def variant_env():
    old = os.environ.get("DPT_U16_VARIANT")
    yield
    if old is None:
        os.environ.pop("DPT_U16_VARIANT", None)
    else:
        os.environ["DPT_U16_VARIANT"] = old


@pytest.mark.parametrize("n", [20, 1000, 70001])
def test_k3_variants_agree(variant_env, n):
    p, o, _ = pr.config("c4b", n)
    r = Checker("oracle").dominant_eigenpair(p, o)
    ref = None
    for v in [0, 2] + ROTATED:
        os.environ["DPT_U16_VARIANT"] = str(v)
        g = P.dominant_eigenpair(p, P.IterationOptions(**o))
        assert int(g.status) == r.status and abs(g.iterations - r.iterations) <= 1, (v, g.status, g.iterations)
        assert abs(g.eigenvalue - r.eigenvalue) <= 1e-10 * max(1.0, abs(r.eigenvalue)), v
        assert np.max(np.abs(g.z_chart - r.z)) < 1e-9, v
        if v in ROTATED:
            if ref is None:
                ref = g
            else:
                assert g.iterations == ref.iterations and np.array_equal(g.z_chart, ref.z_chart), v


@pytest.mark.parametrize("n", [20, 1000, 70001])
def test_complex_u16_pipeline_matches_general_kernel(variant_env, n):
    """Complex data with 16 nonzeros per row: the per-warp pipeline over the
    trip-major CSR copy is bit-identical to the general complex row map (same
    products and sums in CSR order) and matches the reference's complex path."""
    p, o, _ = pr.config("c4b", n)
    p = P.PartitionedProblem(p.d, p.delta, p.lam * (1 + 0.5j))
    outs = {}
    for flag in ("0", "1"):
        os.environ["DPT_CPLX_U16"] = flag
        outs[flag] = P.dominant_eigenpair(p, P.IterationOptions(**o))
    os.environ.pop("DPT_CPLX_U16", None)
    a, b = outs["0"], outs["1"]
    assert int(a.status) == int(b.status) and a.iterations == b.iterations
    assert np.array_equal(a.z_chart, b.z_chart) and a.eigenvalue == b.eigenvalue
    from oracle.bind import ComplexReference, available
    if available("reference"):
        r = ComplexReference().dominant_eigenpair(p, o)
        assert int(b.status) == r.status and abs(b.iterations - r.iterations) <= 1
        if r.status == 0:
            assert abs(b.eigenvalue - r.eigenvalue) <= 1e-10 * max(1.0, abs(r.eigenvalue))


def test_complex_u16_graph_cache_churn():
    """the loop-graph key must cover every buffer a captured launch
    reads.  Solve P1 (complex, 16 per row, device-resident CSR views), then a
    same-n problem from host arrays (churns the context's block cache, so the
    trip-major copies may land elsewhere), then P1 again: the last result is
    bit-identical to the first, and the cache was exercised (hits and misses)."""
    import torch
    ctx = P.Context(0)
    n = 70001
    p1, o, _ = pr.config("c4b", n)
    dv = torch.device("cuda")
    p1 = P.PartitionedProblem(torch.as_tensor(p1.d, device=dv),
                              P.CsrMatrix(n, torch.as_tensor(p1.delta.rowptr, device=dv),
                                          torch.as_tensor(p1.delta.cols, device=dv),
                                          torch.as_tensor(p1.delta.vals, device=dv)),
                              p1.lam * (1 + 0.5j))
    p2, _, _ = pr.config("c4b", n)
    p2 = P.PartitionedProblem(p2.d, P.CsrMatrix(n, p2.delta.rowptr, p2.delta.cols, -p2.delta.vals),
                              p2.lam * (1 - 0.25j))
    io = P.IterationOptions(**o)
    a = P.dominant_eigenpair(p1, io, ctx=ctx)
    P.dominant_eigenpair(p2, io, ctx=ctx)
    P.dominant_eigenpair(p2, io, ctx=ctx)
    b = P.dominant_eigenpair(p1, io, ctx=ctx)
    hits, misses = ctx.graph_stats
    assert misses >= 1 and hits + misses >= 4, (hits, misses)
    assert int(a.status) == int(b.status) and a.iterations == b.iterations
    assert a.eigenvalue == b.eigenvalue
    assert torch.equal(a.z_chart, b.z_chart)  # device-resident inputs -> device-resident outputs
    ctx.close()


@pytest.mark.parametrize("n", [20, 1000, 70001])
def test_unit_start_shortcut_is_bit_identical(variant_env, n):
    """Launch 1 of the row map starts from z_0 = e_row; launch_single_u16_init
    writes z_1 and the partials from the columns alone.  Every output of the
    solve (chart vector, unit vector, eigenvalue, residual, status, iterations,
    trace) equals, bit for bit, the solve whose launch 1 is K3 itself
    (DPT_U16_INIT=0) -- for a rotated and an unrotated K3 variant, the
    dominant pair, a row in the middle of the chart with a trace, and a ramped
    coupling."""
    p, o, _ = pr.config("c4b", n)
    try:
        for v in (16, 0):
            os.environ["DPT_U16_VARIANT"] = str(v)
            outs = {}
            for flag in ("0", "1"):
                os.environ["DPT_U16_INIT"] = flag
                tr = []
                d = P.dominant_eigenpair(p, P.IterationOptions(**o))
                s1 = P.iterate_single(p, n // 2, P.IterationOptions(**o), trace=lambda k, s, m: tr.append((k, s, m)))
                s2 = P.iterate_single(p, n - 1, P.IterationOptions(**o), ramp_alpha=0.5)
                outs[flag] = (d, s1, s2, tr)
            a, b = outs["0"], outs["1"]
            assert a[0].status == b[0].status and a[0].iterations == b[0].iterations, v
            assert a[0].eigenvalue == b[0].eigenvalue and a[0].residual == b[0].residual, v
            assert np.array_equal(a[0].z_chart, b[0].z_chart) and np.array_equal(a[0].z_unit, b[0].z_unit), v
            for q in (1, 2):
                assert a[q].status == b[q].status and a[q].iterations == b[q].iterations, (v, q)
                assert a[q].eigenvalue == b[q].eigenvalue and np.array_equal(a[q].z, b[q].z), (v, q)
            assert a[3] == b[3] and len(a[3]) >= 1, v
    finally:
        os.environ.pop("DPT_U16_INIT", None)
