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
