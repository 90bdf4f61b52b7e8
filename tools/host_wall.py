"""Wall-clock of the public call with HOST (numpy, pageable) inputs and outputs,
best of --reps after one warm-up call, next to the device time of the solve.
The difference is the host<->device traffic of the drop-in boundary."""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2002_12872_b200 as P  # noqa: E402
from paper_2002_12872_b200 import problems as pr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1,c2b,c3,c4,c4b")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
for name in a.configs.split(","):
    p, o, desc = pr.config(name)
    single = name.startswith("c4")
    run = (lambda: P.dominant_eigenpair(p, P.IterationOptions(**o))) if single else \
        (lambda: P.iterate_full(p, P.IterationOptions(**o)))
    r = run()
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        r = run()
        ts.append((time.perf_counter() - t0) * 1e3)
    n = len(p.d)
    h2d = (p.delta.nnz * 12 + (n + 1) * 8 if hasattr(p.delta, "rowptr") else n * n * 8) + n * 8
    d2h = (n * 8 if single else n * n * 8 + 2 * n * 8)
    print(json.dumps({"config": name, "status": P.to_string(r.status), "iterations": r.iterations,
                      "wall_ms": min(ts), "device_ms": r.device_ms, "h2d_MB": h2d / 1e6, "d2h_MB": d2h / 1e6}),
          flush=True)
