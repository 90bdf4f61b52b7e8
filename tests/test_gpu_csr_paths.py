"""GPU: every K2 staging variant against the reference.  The CSR full map
stages R = floor(200 KB / 8n) rows of A per CTA in shared memory (odd-stride
interleaved, bank-aware schedule) and falls back to global-memory gathers when
a row does not fit (n > 25600 real, > 12800 complex).  DPT_CSR_ROWS forces a
smaller R so every variant (R = 0 global, 1, 2 -> stride 3, 3, ...) runs at a
test size; results must match the reference's at the parity bar and each
other bit for bit (the accumulation order does not depend on R)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle.bind import available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not available("reference"), reason="oracle/_ref not built")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2002_12872_b200 as P
from paper_2002_12872_b200 import problems as pr
from paper_2002_12872_b200.dpt import CsrMatrix, PartitionedProblem
cplx = sys.argv[1] == "1"
n = 600
c = pr.csr_sym_bernoulli(n, 11, 0.02)
vals = c.vals + (1j * np.random.default_rng(1).uniform(-0.5, 0.5, c.nnz) if cplx else 0)
lam = 0.01 + (0.005j if cplx else 0)
p = PartitionedProblem(np.arange(n, dtype=float), CsrMatrix(n, c.rowptr, c.cols, vals), lam)
r = P.iterate_full(p)
np.savez(sys.argv[2], a=r.state.a, eig=r.eigenvalues, status=int(r.status), iterations=r.iterations)
"""


@pytest.mark.parametrize("cplx", [0, 1], ids=["real", "complex"])
def test_staging_variants_agree_with_reference(tmp_path, cplx):
    from oracle.bind import ComplexReference
    from paper_2002_12872_b200 import problems as pr
    from paper_2002_12872_b200.dpt import CsrMatrix, PartitionedProblem
    outs = {}
    for rows in ("0", "1", "2", "3", "8"):
        f = str(tmp_path / f"r{rows}.npz")
        env = dict(os.environ, DPT_CSR_ROWS=rows)
        subprocess.run([sys.executable, "-c", SCRIPT, str(cplx), f], cwd=ROOT, env=env, check=True, timeout=300)
        outs[rows] = np.load(f)
    base = outs["8"]
    for rows, z in outs.items():  # identical whatever R is
        assert int(z["status"]) == int(base["status"]) and int(z["iterations"]) == int(base["iterations"])
        assert np.array_equal(z["a"], base["a"]) and np.array_equal(z["eig"], base["eig"]), rows
    n = 600
    c = pr.csr_sym_bernoulli(n, 11, 0.02)
    vals = c.vals + (1j * np.random.default_rng(1).uniform(-0.5, 0.5, c.nnz) if cplx else 0)
    lam = 0.01 + (0.005j if cplx else 0)
    p = PartitionedProblem(np.arange(n, dtype=float), CsrMatrix(n, c.rowptr, c.cols, vals), lam)
    r = ComplexReference().iterate_full(p, {})
    assert r.status == int(base["status"]) and abs(r.iterations - int(base["iterations"])) <= 1
    if r.iterations == int(base["iterations"]) and r.status != 2:
        assert np.max(np.abs(base["a"] - r.a)) < 1e-9
        assert np.max(np.abs(base["eig"] - r.eig) / np.maximum(1.0, np.abs(r.eig))) < 1e-10


INIT_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2002_12872_b200 as P
from paper_2002_12872_b200 import problems as pr
from paper_2002_12872_b200.dpt import CsrMatrix, PartitionedProblem
out = {}
def put(tag, r, tr=None):
    out[tag + ".a"] = r.state.a; out[tag + ".eig"] = r.eigenvalues; out[tag + ".res"] = r.residuals
    out[tag + ".meta"] = np.array([int(r.status), r.iterations, r.step_norm])
    if tr is not None: out[tag + ".trace"] = np.array(tr, dtype=float)
# 1. c3-like (no window: n > 1414), trace on
n = 1600
c = pr.csr_sym_bernoulli(n, 5, 0.01)
p = PartitionedProblem(np.arange(n, dtype=float), c, 0.05)
tr = []
put("plain", P.iterate_full(p, P.IterationOptions(), trace=lambda k, s, m: tr.append((k, s, m))), tr)
# 2. window on (n <= 1414), unsymmetric pattern with explicit diagonal entries of Delta
n = 400
rng = np.random.default_rng(3)
rows = [sorted(set(rng.choice(n, 9, replace=False).tolist()) | ({i} if i % 3 == 0 else set())) for i in range(n)]
rowptr = np.zeros(n + 1, dtype=np.int64); rowptr[1:] = np.cumsum([len(r) for r in rows])
cols = np.concatenate([np.array(r, dtype=np.int32) for r in rows]); vals = rng.standard_normal(len(cols))
c2 = CsrMatrix(n, rowptr, cols, vals)
put("window", P.iterate_full(PartitionedProblem(np.arange(n, dtype=float) * 1.5, c2, 0.03)))
# 3. ramped coupling, 4. exactly two applications, 5. a coupling that diverges, 6. one iteration allowed
put("ramped", P.iterate_ramped(PartitionedProblem(np.arange(n, dtype=float) * 1.5, c2, 0.03), 0.5))
fx = P.iterate_fixed(PartitionedProblem(np.arange(n, dtype=float) * 1.5, c2, 0.03), 2, 0.03)
out["fixed.a"] = np.asarray(fx.a if hasattr(fx, "a") else fx)
put("diverged", P.iterate_full(PartitionedProblem(np.arange(n, dtype=float) * 1.5, c2, 40.0)))
put("budget", P.iterate_full(PartitionedProblem(np.arange(n, dtype=float) * 1.5, c2, 0.03), P.IterationOptions(max_iter=1)))
np.savez(sys.argv[1], **out)
"""


def test_identity_start_shortcut_is_bit_identical(tmp_path):
    """Launch 1 of a CSR solve starts from A_0 = I; launch_csr_init writes A_1, the
    statistics, the residual partials and d_1 without the product.  Every
    output of the solve (iterate, eigenvalues, residuals, status, iterations,
    step norm, trace) must equal, bit for bit, the solve whose launch 1 is K2
    itself (DPT_CSR_INIT=0): full map, trace, window, ramped, fixed, Diverged,
    a one-iteration budget; explicit diagonal entries of Delta."""
    outs = {}
    for init in ("0", "1"):
        f = str(tmp_path / f"init{init}.npz")
        env = dict(os.environ, DPT_CSR_INIT=init)
        subprocess.run([sys.executable, "-c", INIT_SCRIPT, f], cwd=ROOT, env=env, check=True, timeout=600)
        outs[init] = np.load(f)
    assert sorted(outs["0"].files) == sorted(outs["1"].files) and len(outs["0"].files) >= 18
    for k in outs["0"].files:
        assert np.array_equal(outs["0"][k], outs["1"][k], equal_nan=True), k
    assert int(outs["1"]["plain.meta"][0]) == 0 and int(outs["1"]["diverged.meta"][0]) == 2  # Converged / Diverged


def test_unsorted_and_repeated_pairs_take_the_product_path():
    """A CSR whose rows list their columns out of order, or repeat a (row, column)
    pair, is still a valid operator for K2 (a repeated pair adds up).  The
    launch-1 shortcut assumes one entry per pair in increasing order, so the
    upload's order check must route such inputs to K2 as launch 1: results equal
    the canonical CSR's to rounding."""
    import paper_2002_12872_b200 as P
    from paper_2002_12872_b200 import problems as pr
    from paper_2002_12872_b200.dpt import CsrMatrix, PartitionedProblem
    n = 320
    c = pr.csr_sym_bernoulli(n, 4, 0.03)
    d = np.arange(n, dtype=float)
    base = P.iterate_full(PartitionedProblem(d, c, 0.02))
    rp, cols, vals = np.asarray(c.rowptr), np.asarray(c.cols), np.asarray(c.vals)
    # 1. every row's entries reversed
    rc, rv = cols.copy(), vals.copy()
    for i in range(n):
        rc[rp[i]:rp[i + 1]] = cols[rp[i]:rp[i + 1]][::-1]
        rv[rp[i]:rp[i + 1]] = vals[rp[i]:rp[i + 1]][::-1]
    r1 = P.iterate_full(PartitionedProblem(d, CsrMatrix(n, rp, rc, rv), 0.02))
    # 2. the first entry of every non-empty row split into two halves (a repeated pair)
    nrp, ncols, nvals = [0], [], []
    for i in range(n):
        cs, vs = cols[rp[i]:rp[i + 1]].tolist(), vals[rp[i]:rp[i + 1]].tolist()
        if cs:
            cs, vs = [cs[0]] + cs, [vs[0] * 0.5, vs[0] * 0.5] + vs[1:]
        ncols += cs
        nvals += vs
        nrp.append(len(ncols))
    r2 = P.iterate_full(PartitionedProblem(d, CsrMatrix(n, np.array(nrp, dtype=np.int64), np.array(ncols, dtype=np.int32),
                                                        np.array(nvals)), 0.02))
    for r in (r1, r2):
        assert r.status == base.status and r.iterations == base.iterations
        assert np.max(np.abs(r.state.a - base.state.a)) < 1e-12
        assert np.max(np.abs(r.eigenvalues - base.eigenvalues)) < 1e-10
