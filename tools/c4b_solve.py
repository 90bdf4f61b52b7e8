import sys; sys.path.insert(0, ".")
import torch
import paper_2002_12872_b200 as P
from paper_2002_12872_b200 import problems as pr
p, o, _ = pr.config("c4b")
dev = torch.device("cuda")
pd = P.PartitionedProblem(torch.as_tensor(p.d, device=dev), P.CsrMatrix(len(p.d), torch.as_tensor(p.delta.rowptr, device=dev), torch.as_tensor(p.delta.cols, device=dev), torch.as_tensor(p.delta.vals, device=dev)), p.lam)
for _ in range(2):
    r = P.dominant_eigenpair(pd, P.IterationOptions(**o))
print(r.iterations, r.device_ms)
