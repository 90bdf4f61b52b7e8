"""GPU: K2's SELL image under every schedule (0 dense packing, 1 CSR-order bank
greedy, 2 free-order bank auction -- the default) with and without the
bank-balancing column relabelling (one and three local-search passes), on
patterns that stress them: a uniform
random pattern, ragged rows (empty rows, a few rows 30x longer than the rest,
a length that is not a multiple of 32), and a pattern whose columns all fall
into a few banks.  Each run must meet the parity bar against the reference's
own iterate_full (same status, iterations +-1, eigenvalues 1e-10 relative,
eigenvectors 1e-9); runs of one pattern agree with each other to rounding."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle.bind import available
from paper_2002_12872_b200.dpt import CsrMatrix, PartitionedProblem

from helpers import eig_rel_err

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not available("reference"), reason="oracle/_ref not built")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2002_12872_b200 as P
from paper_2002_12872_b200.dpt import CsrMatrix, PartitionedProblem
z = np.load(sys.argv[1])
p = PartitionedProblem(z["d"], CsrMatrix(int(z["d"].shape[0]), z["rowptr"], z["cols"], z["vals"]), float(z["lam"]))
r = P.iterate_full(p)
np.savez(sys.argv[2], a=r.state.a, eig=r.eigenvalues, status=int(r.status), iterations=r.iterations)
"""


def _csr_from_sets(n, rows, rng):
    rowptr = np.zeros(n + 1, dtype=np.int64)
    cols, vals = [], []
    for i in range(n):
        c = np.array(sorted(rows[i]), dtype=np.int32)
        cols.append(c)
        vals.append(rng.standard_normal(len(c)))
        rowptr[i + 1] = rowptr[i] + len(c)
    return CsrMatrix(n, rowptr, np.concatenate(cols).astype(np.int32), np.concatenate(vals))


def _pattern(kind):
    rng = np.random.default_rng({"uniform": 21, "ragged": 22, "banked": 23}[kind])
    if kind == "uniform":
        n = 640
        rows = [set(rng.choice(n, 12, replace=False).tolist()) - {i} for i in range(n)]
    elif kind == "ragged":
        n = 1000  # not a multiple of 32
        rows = []
        for i in range(n):
            if i % 97 == 0:
                rows.append(set())  # empty rows
            elif i % 211 == 5:
                rows.append(set(rng.choice(n, 300, replace=False).tolist()) - {i})  # long rows
            else:
                rows.append(set(rng.choice(n, int(rng.integers(1, 20)), replace=False).tolist()) - {i})
    else:  # every column in banks 0..2 (col mod 16 < 3): the schedule's worst case
        n = 512
        pool = np.array([k for k in range(n) if k % 16 < 3])
        rows = [set(rng.choice(pool, 10, replace=False).tolist()) - {i} for i in range(n)]
    return n, _csr_from_sets(n, rows, rng)


@pytest.mark.parametrize("kind", ["uniform", "ragged", "banked"])
def test_schedules_and_relabelling_match_reference(tmp_path, kind):
    from oracle.bind import ComplexReference
    n, csr = _pattern(kind)
    lam = 0.02
    d = np.arange(n, dtype=float)
    f = str(tmp_path / "p.npz")
    np.savez(f, d=d, rowptr=csr.rowptr, cols=csr.cols, vals=csr.vals, lam=lam)
    ref = ComplexReference().iterate_full(PartitionedProblem(d, csr, lam), {})
    outs = {}
    for sched in ("0", "1", "2"):
        for relabel in ("0", "1"):
            if sched != "2" and relabel == "1":
                continue  # the relabelling only serves the free-order schedule
            o = str(tmp_path / f"s{sched}r{relabel}.npz")
            env = dict(os.environ, DPT_SELL_SCHED=sched, DPT_SELL_RELABEL=relabel)
            subprocess.run([sys.executable, "-c", SCRIPT, f, o], cwd=ROOT, env=env, check=True, timeout=300)
            g = np.load(o)
            outs[(sched, relabel)] = g
            assert int(g["status"]) == ref.status, (sched, relabel, int(g["status"]), ref.status)
            assert abs(int(g["iterations"]) - ref.iterations) <= 1, (sched, relabel)
            if int(g["iterations"]) == ref.iterations and ref.status != 2:
                assert np.max(np.abs(g["a"] - ref.a)) < 1e-9, (sched, relabel)
                assert eig_rel_err(g["eig"], ref.eig) < 1e-10, (sched, relabel)
    # three local-search passes of the relabelling instead of the default one (DPT_SELL_PASSES)
    o = str(tmp_path / "s2r1p3.npz")
    env = dict(os.environ, DPT_SELL_SCHED="2", DPT_SELL_RELABEL="1", DPT_SELL_PASSES="3")
    subprocess.run([sys.executable, "-c", SCRIPT, f, o], cwd=ROOT, env=env, check=True, timeout=300)
    g = np.load(o)
    outs[("2", "1p3")] = g
    assert int(g["status"]) == ref.status and abs(int(g["iterations"]) - ref.iterations) <= 1
    base = outs[("2", "1")]
    for key, g in outs.items():
        if int(g["iterations"]) == int(base["iterations"]) and int(base["status"]) != 2:
            assert np.max(np.abs(g["a"] - base["a"])) < 1e-12, key


RELABEL_EDGE = r"""
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2002_12872_b200 as P
from paper_2002_12872_b200 import problems as pr
from paper_2002_12872_b200.dpt import PartitionedProblem
from oracle.bind import Checker
for n in (64, 65, 96, 127, 128, 129, 200, 257):
    c = pr.csr_sym_bernoulli(n, 100 + n, 0.08)
    p = PartitionedProblem(np.arange(n, dtype=float), c, 0.02)
    g = P.iterate_full(p)
    r = Checker("oracle").iterate_full(p, {})
    assert int(g.status) == r.status and abs(g.iterations - r.iterations) <= 1, n
    assert np.max(np.abs(g.state.a - r.a)) < 1e-9, n
"""


@pytest.mark.parametrize("passes", ["1", "3"])
def test_relabel_batch_boundaries(passes):
    """The relabelling walks the columns in batches of 64, software-pipelined
    (the next batch prefetched while the current one is evaluated): sizes of
    exactly one batch (n = 64: the next batch is the same columns, re-read after
    this batch's writes), one column more, a partial last batch, several
    batches -- each against the oracle, with one and three passes."""
    env = dict(os.environ, DPT_SELL_PASSES=passes)
    subprocess.run([sys.executable, "-c", RELABEL_EDGE], cwd=ROOT, env=env, check=True, timeout=300)
