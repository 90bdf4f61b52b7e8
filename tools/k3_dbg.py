"""K3 variant debug: one step_single per variant on the same z, bitwise compare."""
import os, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2002_12872_b200 as P
from paper_2002_12872_b200 import problems as pr
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
p, o, _ = pr.config("c4b", n)
rng = np.random.default_rng(5)
z = rng.standard_normal(n) * 1e-3
z[n - 1] = 1.0
outs = {}
for v in [1, 3, 4, 5, 6, 8, 10]:
    os.environ["DPT_U16_VARIANT"] = str(v)
    outs[v] = P.step_single(z, n - 1, p, p.lam)
    d = outs[v] != outs[1]
    print(v, "diff count", int(d.sum()), "first idx", np.nonzero(d)[0][:10])
