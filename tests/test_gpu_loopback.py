"""GPU: the world > 1 CUDA path on ONE device.  Two to eight contexts on
device 0 form a loopback group (dpt_ctx_set_loopback, test-only): each rank
is driven by its own host thread through the public calls, so the real sharded
code runs -- shard_rows -> per-rank step kernel on its row block -> max-
allreduce of the statistics -> decide -> cycle -> gather of the rows and
read-offs (solver.cu).  The collectives are in-process (host rendezvous +
stream-event dependencies + device copies; no kernel waits on another rank's
kernel).  The rows of A evolve independently and the statistics are maxima, so
the sharded solve must equal the unsharded one BIT FOR BIT, and the oracle
within the north_star tolerances."""
import threading

import numpy as np
import pytest

import paper_2002_12872_b200 as P
from oracle.bind import Checker
from paper_2002_12872_b200 import problems as pr

from helpers import assert_full_parity

pytestmark = pytest.mark.gpu
O = Checker("oracle")


def run_ranks(world, fn):
    """fn(ctx) on `world` loopback ranks, one thread each; returns the results."""
    ctxs = [P.Context(0) for _ in range(world)]
    P.Context.set_loopback(ctxs)
    out, errs = [None] * world, [None] * world

    def one(r):
        try:
            out[r] = fn(ctxs[r])
        except Exception as e:  # noqa: BLE001 -- re-raised below
            errs[r] = e

    ths = [threading.Thread(target=one, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=600)
    for c in ctxs:
        c.close()
    for e in errs:
        if e is not None:
            raise e
    return out


def assert_same_report(g, h):
    assert int(g.status) == int(h.status) and g.iterations == h.iterations
    assert g.step_norm == h.step_norm or (np.isnan(g.step_norm) and np.isnan(h.step_norm))
    assert np.array_equal(g.state.a, h.state.a, equal_nan=True)
    assert np.array_equal(g.eigenvalues, h.eigenvalues, equal_nan=True)
    assert np.array_equal(g.residuals, h.residuals, equal_nan=True)


@pytest.mark.parametrize("name,n,world", [("c1", 300, 2), ("c1", 301, 3), ("c1", 301, 4), ("c2b", 1024, 2),
                                          ("c2", 256, 2), ("c2b", 777, 8), ("c3", 512, 2), ("c3", 515, 3)])
def test_sharded_solve_equals_unsharded(name, n, world):
    p, o, _ = pr.config(name, n)
    io = P.IterationOptions(**o)
    h = P.iterate_full(p, io)  # single device
    got = run_ranks(world, lambda ctx: P.iterate_full(p, io, ctx=ctx))
    for g in got:  # every rank returns the gathered result
        assert_same_report(g, h)
    r = O.iterate_full(p, o)
    assert_full_parity(got[0], r.status, r.iterations, r.a, r.eig, r.res)


def test_sharded_cycle_window_and_trace():
    """c1 sizes keep the cycle window on (n <= 1414): the cycle flags of every
    rank's rows are combined by the allreduce; the trace is the same on every
    rank and equals the unsharded one."""
    p = pr.two_by_two(0.88)
    h = P.iterate_full(p)
    got = run_ranks(2, lambda ctx: P.iterate_full(p, ctx=ctx))
    assert h.status == P.ConvergenceStatus.BoundedNonConverged
    for g in got:
        assert_same_report(g, h)
    p, o, _ = pr.config("c1", 200)
    tr_h = []
    P.iterate_full(p, P.IterationOptions(**o), trace=lambda k, s, m: tr_h.append((k, s, m)))

    def traced(ctx):
        t = []
        P.iterate_full(p, P.IterationOptions(**o), trace=lambda k, s, m: t.append((k, s, m)), ctx=ctx)
        return t

    for t in run_ranks(2, traced):
        assert t == tr_h


def test_sharded_fixed_and_ramped():
    p, o, _ = pr.config("c1", 256)
    a = run_ranks(2, lambda ctx: P.iterate_fixed(p, 3, p.lam, ctx=ctx))
    b = P.iterate_fixed(p, 3, p.lam)
    for x in a:
        assert np.array_equal(x, b)
    g = run_ranks(2, lambda ctx: P.iterate_ramped(p, 0.5, P.IterationOptions(**o), ctx=ctx))
    h = P.iterate_ramped(p, 0.5, P.IterationOptions(**o))
    for x in g:
        assert_same_report(x, h)


def test_sharded_plan_steps():
    """The bench's fixed-step Plan on 2 ranks: the gathered iterate after k
    steps equals the single-device plan's."""
    p, _, _ = pr.config("c2", 512)

    def steps(ctx):
        pl = P.Plan(p, ctx=ctx)
        pl.begin()
        pl.steps(3)
        a = pl.read()
        pl.close()
        return a

    single = steps(None)
    for a in run_ranks(2, steps):
        assert np.array_equal(a, single)


def test_row_map_replicas():
    """The single-vector mode does not shard (one SpMV chain): with a
    communicator every rank runs the whole row map as a replica, the
    statistics all-reduce over identical values, and every rank returns the
    single-device answer bit for bit ("replicas only")."""
    p, o, _ = pr.config("c4b", 20000)
    io = P.IterationOptions(**o)
    h = P.dominant_eigenpair(p, io)
    for g in run_ranks(2, lambda ctx: P.dominant_eigenpair(p, io, ctx=ctx)):
        assert int(g.status) == int(h.status) and g.iterations == h.iterations and g.row == h.row
        assert g.eigenvalue == h.eigenvalue and np.array_equal(g.z_chart, h.z_chart)
