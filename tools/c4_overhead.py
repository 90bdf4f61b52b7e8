"""Per-iteration device time of the row-map solve (c4 / c4b) through the
public call with device-resident inputs, next to the plan-step time (K3 alone):
the difference is the fold / decision / cycle pre-check of the device loop."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2002_12872_b200 as P  # noqa: E402
from paper_2002_12872_b200 import problems as pr  # noqa: E402

dev = torch.device("cuda")
for name in ("c4", "c4b"):
    p, o, _ = pr.config(name)
    n = len(p.d)
    pd = P.PartitionedProblem(torch.as_tensor(p.d, device=dev),
                              P.CsrMatrix(n, torch.as_tensor(p.delta.rowptr, device=dev),
                                          torch.as_tensor(p.delta.cols, device=dev),
                                          torch.as_tensor(p.delta.vals, device=dev)), p.lam)
    best = None
    for _ in range(5):
        r = P.dominant_eigenpair(pd, P.IterationOptions(**o))
        best = r.device_ms if best is None else min(best, r.device_ms)
    plan = P.Plan(pd, single=True, row=n - 1)
    plan.begin()
    plan.steps(3)
    torch.cuda.synchronize()
    kms = plan.steps(20, time_kernel=True) / 20
    plan.close()
    print(json.dumps({"config": name, "status": P.to_string(r.status), "iterations": r.iterations, "solve_device_ms_best5": best,
                      "per_iteration_us": best * 1e3 / r.iterations, "plan_step_kernel_us": kms * 1e3}), flush=True)
