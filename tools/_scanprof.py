import sys, time
sys.path.insert(0, ".")
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2002_12872_b200 as P
from paper_2002_12872_b200 import problems as pr
from paper_2002_12872_b200.dpt import IterationOptions, PartitionedProblem, ScanGrid, ScanMode
for name, p, mode, row, g in [("2x2", pr.two_by_two(1.0), "Full", 0, ScanGrid(-1.2, 1.2, -1.0, 1.0, 512, 512)),
                              ("n6", PartitionedProblem(*pr.random_uniform(6, 3), 0.0), "Full", 0, ScanGrid(-0.4, 0.4, -0.3, 0.3, 512, 512))]:
    o = IterationOptions(max_iter=300)
    P.scan_domain(p, g, ScanMode(mode, row), o)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        t0 = time.perf_counter()
        P.scan_domain(p, g, ScanMode(mode, row), o)
        t1 = time.perf_counter()
    ks = [(e.name[:50], e.time_range.elapsed_us()) for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    print(name, "wall_ms", round((t1 - t0) * 1e3, 2), ks[:8])
