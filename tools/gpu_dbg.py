import sys, os
sys.path.insert(0, ".")
import numpy as np
import paper_2002_12872_b200 as P
from paper_2002_12872_b200 import problems as pr
for name, n, win in [("c1", 64, 0), ("c1", 64, 16), ("c3", 64, 0)]:
    p, o, desc = pr.config(name, n)
    o["cycle_window"] = win
    try:
        g = P.iterate_full(p, P.IterationOptions(**o))
        print(name, n, win, P.to_string(g.status), g.iterations, flush=True)
    except Exception as e:
        print(name, n, win, "ERR", e, flush=True)
        break
