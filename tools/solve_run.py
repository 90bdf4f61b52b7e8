"""One solve of a config (for launch lists under ncu)."""
import argparse
import sys

sys.path.insert(0, ".")
import paper_2002_12872_b200 as P  # noqa: E402
from paper_2002_12872_b200 import problems as pr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--n", type=int, default=None)
a = ap.parse_args()
p, o, desc = pr.config(a.config, a.n)
if a.config.startswith("c4"):
    r = P.dominant_eigenpair(p, P.IterationOptions(**o))
else:
    r = P.iterate_full(p, P.IterationOptions(**o))
print(desc, P.to_string(r.status), r.iterations, r.device_ms)
