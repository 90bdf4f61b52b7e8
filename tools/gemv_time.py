"""Row map with a DENSE Delta (the GEMV flavour of the single-vector mode):
event-timed step kernel vs the HBM roofline.  Development / profiles helper."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2002_12872_b200 as P  # noqa: E402
from paper_2002_12872_b200 import problems as pr  # noqa: E402

HBM = 6547.2
for n in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8192,16384,32768").split(",")]:
    dev = torch.device("cuda")
    d = torch.as_tensor(pr.theta_linear(n, 1.0 / n), device=dev)
    g = torch.Generator(device="cuda").manual_seed(7)
    delta = torch.randn((n, n), dtype=torch.float64, device=dev, generator=g)
    delta.fill_diagonal_(0.0)
    p = P.PartitionedProblem(d, delta, 0.5 / n ** 0.5)
    plan = P.Plan(p, single=True, row=n - 1)
    plan.begin()
    plan.steps(3)
    torch.cuda.synchronize()
    k = 20
    kms = plan.steps(k, time_kernel=True) / k
    plan.close()
    byts = 8.0 * n * n + 8 * 3 * n  # Delta once + z, theta, z'
    print(json.dumps({"n": n, "kernel_ms": kms, "gbs": byts / (kms * 1e-3) / 1e9,
                      "hbm_frac": byts / (kms * 1e-3) / 1e9 / HBM}))
    del delta
    torch.cuda.empty_cache()
