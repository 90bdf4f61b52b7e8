"""Generates tests/golden/*.npz from the REFERENCE implementation itself
(oracle/_ref/libdynspec_ref.so = /root/reference/proj/src compiled by
oracle/Makefile).  Run in the build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py
    python tests/golden/make_golden.py c3full     # c3 at n = 8192 (~2 min)
    python tests/golden/make_golden.py c2bfull    # c2b at n = 4096 (~20 min)

The fixtures are small (n <= 96) so they travel with the repo; the tests check
both the C restatement and the CUDA path against them.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.bind import Checker  # noqa: E402
from paper_2002_12872_b200 import problems as pr  # noqa: E402
from paper_2002_12872_b200.dpt import PartitionedProblem  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def cases():
    out = []
    for name, n in [("c1", 48), ("c1", 96), ("c2", 64), ("c2b", 80), ("c3", 96)]:
        p, o, _ = pr.config(name, n)
        out.append((f"{name}_n{n}", p, o))
    t, a = pr.random_uniform(7, 17)
    out.append(("random_uniform_n7_lam0.03", PartitionedProblem(t, a, 0.03), {}))
    t, a = pr.oscillator(24)
    out.append(("oscillator_n24_lam0.5", PartitionedProblem(t, a, 0.5), {}))
    out.append(("two_by_two_lam0.88", pr.two_by_two(0.88), {}))
    return out


def main():
    R = Checker("reference")
    for name, p, o in cases():
        r = R.iterate_full(p, o, trace=True)
        rec = dict(d=p.d, lam=p.lam, status=r.status, iterations=r.iterations, step_norm=r.step_norm, a=r.a,
                   eig=r.eig, res=r.res, trace_step=r.trace_step, trace_res=r.trace_res,
                   opts=np.array([o.get("tol", 1e-12), o.get("max_iter", 10000)]))
        if hasattr(p.delta, "rowptr"):
            rec.update(rowptr=p.delta.rowptr, cols=p.delta.cols, vals=p.delta.vals)
        else:
            rec.update(delta=p.delta)
        a2 = R.iterate_fixed(p, 2, p.lam)[1]
        rec.update(fixed2=a2)
        np.savez_compressed(os.path.join(OUT, f"full_{name}.npz"), **rec)
        print(name, r.status, r.iterations)
    for name, n in [("c4", 2048), ("c4b", 4096)]:
        p, o, _ = pr.config(name, n)
        r = R.dominant_eigenpair(p, o)
        np.savez_compressed(os.path.join(OUT, f"dominant_{name}_n{n}.npz"), d=p.d, lam=p.lam,
                            rowptr=p.delta.rowptr, cols=p.delta.cols, vals=p.delta.vals, status=r.status,
                            iterations=r.iterations, eigenvalue=r.eigenvalue, residual=r.residual, z=r.z,
                            z_unit=r.z_unit, row=r.row, step_norm=r.step_norm)
        print(name, n, r.status, r.iterations)


C3_ROWS = ((0, 64), (4000, 4064))


def c3_full():
    """BASELINE configs[2] at its full size (n = 8192 CSR, ~92 s in the
    reference): status, iterations, all eigenvalues and residuals, and two
    64-row blocks of the final eigenvector matrix.  The inputs are regenerated
    by the tests from the recipe; their fingerprint is stored to pin them."""
    R = Checker("reference")
    p, o, _ = pr.config("c3")
    r = R.iterate_full(p, o)
    rec = dict(status=r.status, iterations=r.iterations, step_norm=r.step_norm, eig=r.eig, res=r.res,
               nnz=p.delta.nnz, vals_sum=np.sum(p.delta.vals), cols_sum=np.sum(p.delta.cols.astype(np.int64)),
               lam=p.lam)
    for a, b in C3_ROWS:
        rec[f"a_{a}_{b}"] = r.a[a:b]
    np.savez_compressed(os.path.join(OUT, "c3full_n8192.npz"), **rec)
    print("c3 full", r.status, r.iterations)


C2B_ROWS = ((0, 64), (2000, 2064))


def c2b_full():
    """The bench family at its full size: c2b (BASELINE configs[1] with theta_i
    = i, the converging companion; n = 4096 dense unsymmetric, ~20 min in the
    reference).  Status, iterations, all eigenvalues and residuals, two 64-row
    blocks of the eigenvector matrix, and the inputs' fingerprint."""
    R = Checker("reference")
    p, o, _ = pr.config("c2b")
    r = R.iterate_full(p, o)
    rec = dict(status=r.status, iterations=r.iterations, step_norm=r.step_norm, eig=r.eig, res=r.res,
               delta_sum=np.sum(p.delta), delta_sq=np.sum(p.delta * p.delta), lam=p.lam)
    for a, b in C2B_ROWS:
        rec[f"a_{a}_{b}"] = r.a[a:b]
    np.savez_compressed(os.path.join(OUT, "c2bfull_n4096.npz"), **rec)
    print("c2b full", r.status, r.iterations)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "c3full":
        c3_full()
    elif len(sys.argv) > 1 and sys.argv[1] == "c2bfull":
        c2b_full()
    else:
        main()
