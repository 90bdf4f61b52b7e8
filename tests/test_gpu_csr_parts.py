"""GPU: K2's split staging (csr_step_parts_kernel, sparse_step.cu).  The
image schedules each lane's entries range by range of staged positions, and
every kernel that streams the image accumulates in that order, so the split
kernel (ranges staged one after the other, partial dots parked in L2) must
equal the whole-row kernel (DPT_CSR_ROWS forces it) BIT FOR BIT over the same
image, and the oracle within the north_star tolerances.  Sizes include ragged
row blocks and the BASELINE c3 size (which uses 2 ranges by default)."""
import os

import numpy as np
import pytest

import paper_2002_12872_b200 as P
from oracle.bind import Checker
from paper_2002_12872_b200 import problems as pr

from helpers import assert_full_parity

pytestmark = pytest.mark.gpu
O = Checker("oracle")


@pytest.fixture
def env():
    keys = ("DPT_CSR_PARTS", "DPT_CSR_ROWS")
    old = {k: os.environ.get(k) for k in keys}
    yield os.environ
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def solve(p, o, **knobs):
    for k in ("DPT_CSR_PARTS", "DPT_CSR_ROWS"):
        os.environ.pop(k, None)
    os.environ.update({k: str(v) for k, v in knobs.items()})
    return P.iterate_full(p, P.IterationOptions(**o))


@pytest.mark.parametrize("n,parts", [(300, 2), (515, 2), (515, 3), (1024, 4), (2000, 2)])
def test_parts_equal_whole_rows(env, n, parts):
    p, o, _ = pr.config("c3", n)
    split = solve(p, o, DPT_CSR_PARTS=parts)
    for rows in (1, 2):
        whole = solve(p, o, DPT_CSR_PARTS=parts, DPT_CSR_ROWS=rows)
        assert int(whole.status) == int(split.status) and whole.iterations == split.iterations
        assert np.array_equal(whole.state.a, split.state.a), rows
        assert np.array_equal(whole.eigenvalues, split.eigenvalues)
    r = O.iterate_full(p, o)
    assert_full_parity(split, r.status, r.iterations, r.a, r.eig, r.res)


def test_parts_fixed_steps_c3_size(env):
    """c3 at n = 8192: the default (2 ranges, 6 rows per CTA) against the
    whole-row kernel over the same image, 3 map applications."""
    p, _, _ = pr.config("c3")
    os.environ.pop("DPT_CSR_ROWS", None)
    os.environ.pop("DPT_CSR_PARTS", None)
    a = P.iterate_fixed(p, 3, p.lam)
    os.environ["DPT_CSR_ROWS"] = "3"
    b = P.iterate_fixed(p, 3, p.lam)
    assert np.array_equal(a, b)
    rows = slice(4000, 4008)
    a2 = P.iterate_fixed(p, 2, p.lam)
    want = O.step_rows(p, 4000, a2[rows], p.lam)
    assert np.max(np.abs(a[rows] - want)) < 1e-12
