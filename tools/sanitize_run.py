"""Small solves through every hot kernel, for compute-sanitizer (racecheck /
synccheck / memcheck): K1 (dense_step_kernel, real and complex), K2
(csr_step_kernel), K3 (single_u16w_kernel, real and complex per-warp
pipelines), fold / decide / cycle, the loopback-free sharded path is not
exercised here; the homotopy's GEMM / cluster LU (linalg.cu).  Host-driven
launches (DPT_GRAPH_LOOP=0) so every kernel is a plain launch."""
import os
import sys

os.environ["DPT_GRAPH_LOOP"] = "0"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2002_12872_b200 as P  # noqa: E402
from paper_2002_12872_b200 import problems as pr  # noqa: E402

p, o, _ = pr.config("c1", 160)
g = P.iterate_full(p, P.IterationOptions(**o))
print("K1 real", P.to_string(g.status), g.iterations)
pc = P.PartitionedProblem(p.d, p.delta, p.lam * (1 + 0.5j))
g = P.iterate_full(pc, P.IterationOptions(**o))
print("K1 complex", P.to_string(g.status), g.iterations)
p, o, _ = pr.config("c2b", 2048)
g = P.iterate_fixed(p, 2, p.lam)
print("K1 128x64 tiles", g.shape)
p, o, _ = pr.config("c3", 300)
g = P.iterate_full(p, P.IterationOptions(**o))
print("K2", P.to_string(g.status), g.iterations)
p, o, _ = pr.config("c4b", 8192)
g = P.dominant_eigenpair(p, P.IterationOptions(**o))
print("K3", P.to_string(g.status), g.iterations)
pc = P.PartitionedProblem(p.d, p.delta, p.lam * (1 + 0.5j))
g = P.dominant_eigenpair(pc, P.IterationOptions(**o))
print("K3 complex", P.to_string(g.status), g.iterations)
rng = np.random.default_rng(1)
a = rng.standard_normal((100, 100)) + 10 * np.eye(100)
x = P.solve_linear_multi(a, rng.standard_normal((100, 3)))
print("LU", float(np.max(np.abs(x))))
print("GEMM", float(np.max(np.abs(P.matmul_dense(a, a)))))
