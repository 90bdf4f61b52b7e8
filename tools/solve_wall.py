"""Wall-clock of repeated solves (host API, device-resident inputs): graph-loop
vs chunked driver comparisons (dev helper)."""
import argparse
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2002_12872_b200 as P  # noqa: E402
from paper_2002_12872_b200 import problems as pr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1,c4,c4b,c2b")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
dev = torch.device("cuda")
for name in a.configs.split(","):
    p, o, desc = pr.config(name)
    if hasattr(p.delta, "rowptr"):
        delta = P.CsrMatrix(len(p.d), torch.as_tensor(p.delta.rowptr, device=dev),
                            torch.as_tensor(p.delta.cols, device=dev), torch.as_tensor(p.delta.vals, device=dev))
    else:
        delta = torch.as_tensor(p.delta, device=dev)
    pd = P.PartitionedProblem(torch.as_tensor(p.d, device=dev), delta, p.lam)
    single = name.startswith("c4")
    run = (lambda: P.dominant_eigenpair(pd, P.IterationOptions(**o))) if single else \
        (lambda: P.iterate_full(pd, P.IterationOptions(**o)))
    ts = []
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = run()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{name}: {P.to_string(r.status)} {r.iterations} wall_ms first={ts[0]:.3f} best={min(ts):.3f} "
          f"device_ms={r.device_ms:.3f}", flush=True)
