"""Timings of the library-free device linear algebra (csrc/linalg.cu) and the
device homotopy_solve built on it: GEMM TFLOP/s (device-resident via the
homotopy's own use is internal, so the public matmul_dense is timed with host
arrays AND its kernel share from a kineto trace), LU solve, homotopy c1 / c2b."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2002_12872_b200 as P  # noqa: E402
from paper_2002_12872_b200 import problems as pr  # noqa: E402


def kernels(fn):
    fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    out = {}
    for e in prof.events():
        if e.device_type != torch.autograd.DeviceType.CUDA or "Memcpy" in e.name or "Memset" in e.name:
            continue
        import re
        m = re.search(r"(\w+_kernel)", e.name)
        k = m.group(1) if m else e.name[:40]
        c, t = out.get(k, (0, 0.0))
        out[k] = (c + 1, t + e.time_range.elapsed_us())
    return {k: {"n": c, "us": round(t, 1)} for k, (c, t) in out.items()}


rng = np.random.default_rng(0)
for n in (1024, 4096):
    a, b = rng.standard_normal((n, n)), rng.standard_normal((n, n))
    ks = kernels(lambda: P.matmul_dense(a, b))
    g = [v for k, v in ks.items() if "gemm_nt" in k][0]
    print(json.dumps({"gemm_n": n, "kernel_us": g["us"], "tflops": 2 * n ** 3 / (g["us"] * 1e-6) / 1e12}), flush=True)
    m = a + 3 * np.sqrt(n) * np.eye(n)
    t0 = time.perf_counter()
    P.solve_linear_multi(m, b)
    wall = time.perf_counter() - t0
    ks = kernels(lambda: P.solve_linear_multi(m, b))
    tot = sum(v["us"] for v in ks.values())
    print(json.dumps({"solve_n": n, "nrhs": n, "wall_ms_host_arrays": wall * 1e3, "device_kernel_ms": tot / 1e3,
                      "kernels": ks}), flush=True)
for name, n in (("c1", 1024), ("c2b", 4096)):
    p, o, _ = pr.config(name, n)
    P.homotopy_solve(p, 2, P.IterationOptions(**o))
    t0 = time.perf_counter()
    h = P.homotopy_solve(p, 2, P.IterationOptions(**o))
    wall = time.perf_counter() - t0
    print(json.dumps({"homotopy": name, "n": n, "stages": 2, "status": P.to_string(h.status),
                      "iterations": h.iterations, "wall_ms": wall * 1e3}), flush=True)
