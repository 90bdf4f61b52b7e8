"""Quick GPU parity probe (development helper): CUDA path vs the C restatement."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2002_12872_b200 as P
from paper_2002_12872_b200 import problems as pr
from oracle.bind import Checker

O = Checker("oracle")
cases = [("c1", 64), ("c1", 200), ("c1", 1024), ("c2", 256), ("c2b", 512), ("c3", 512), ("c3", 2048), ("c2b", 2048)]
for name, n in cases:
    p, o, desc = pr.config(name, n)
    t = time.time(); g = P.iterate_full(p, P.IterationOptions(**o)); tg = time.time() - t
    t = time.time(); r = O.iterate_full(p, o); tr = time.time() - t
    fin = np.isfinite(r.eig)
    de = np.max(np.abs(g.eigenvalues[fin] - r.eig[fin]) / np.maximum(1, np.abs(r.eig[fin]))) if fin.any() else 0
    da = np.nanmax(np.abs(g.state.a - r.a)) if r.status != 2 else float("nan")
    print(f"{name} n={n}: gpu {P.to_string(g.status)} {g.iterations} step {g.step_norm:.3e} | ref {r.status} {r.iterations} step {r.step_norm:.3e} | eig rel {de:.2e} A {da:.2e} res max {np.nanmax(g.residuals):.2e}/{np.nanmax(r.res):.2e} | {g.device_ms:.2f} ms gpu, {tr:.2f}s cpu", flush=True)
for name, n in [("c4", 4096), ("c4b", 65536)]:
    p, o, desc = pr.config(name, n)
    g = P.dominant_eigenpair(p, P.IterationOptions(**o))
    r = O.dominant_eigenpair(p, o)
    print(f"{name} n={n}: gpu {P.to_string(g.status)} {g.iterations} eig {g.eigenvalue:.15g} | ref {r.status} {r.iterations} eig {r.eigenvalue:.15g} | z {np.nanmax(np.abs(g.z_chart - r.z)):.2e} zu {np.nanmax(np.abs(g.z_unit - r.z_unit)):.2e}", flush=True)
