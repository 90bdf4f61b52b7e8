"""GPU: the sharded (multi-GPU) code path on one device.  A 1-rank NCCL
communicator switches the solver to its collective path -- the per-iteration
ncclAllReduce(MAX) of the statistics between the fold and a separate decision
kernel, and the ncclAllGather of the final rows / read-offs -- so the NCCL
plumbing runs for real; results must equal the single-device path and the
oracle.  (Multi-rank sharding logic itself: tests/test_host.py, gloo.)"""
import numpy as np
import pytest

import paper_2002_12872_b200 as P
from oracle.bind import Checker
from paper_2002_12872_b200 import problems as pr

from helpers import assert_full_parity

pytestmark = pytest.mark.gpu
O = Checker("oracle")


@pytest.fixture(scope="module")
def comm_ctx():
    ctx = P.Context(0)
    try:
        ctx.set_comm(0, 1, P.Context.nccl_unique_id())
    except P.DeviceError as e:  # libnccl.so.2 must be loadable on the GPU box
        pytest.fail(f"NCCL path unavailable: {e}")
    yield ctx
    ctx.close()


@pytest.mark.parametrize("name,n", [("c1", 300), ("c2", 256), ("c2b", 2048), ("c3", 512)])
def test_collective_path_matches_oracle(comm_ctx, name, n):
    p, o, _ = pr.config(name, n)
    g = P.iterate_full(p, P.IterationOptions(**o), ctx=comm_ctx)
    r = O.iterate_full(p, o)
    assert_full_parity(g, r.status, r.iterations, r.a, r.eig, r.res)
    h = P.iterate_full(p, P.IterationOptions(**o))  # single-device path, same answer
    assert int(h.status) == int(g.status) and h.iterations == g.iterations
    if int(g.status) != 2:
        assert np.array_equal(h.state.a, g.state.a)
        assert np.array_equal(h.eigenvalues, g.eigenvalues)


def test_collective_path_cycle_and_fixed(comm_ctx):
    g = P.iterate_full(pr.two_by_two(0.88), ctx=comm_ctx)
    assert g.status == P.ConvergenceStatus.BoundedNonConverged
    p, o, _ = pr.config("c1", 200)
    a = P.iterate_fixed(p, 3, p.lam, ctx=comm_ctx)
    rc, b = O.iterate_fixed(p, 3, p.lam)
    assert np.max(np.abs(a - b)) < 1e-12
