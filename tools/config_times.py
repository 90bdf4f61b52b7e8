"""Per-config device timings (fixed steps through a Plan) + time-to-status of the
full solve, with roofline fractions.  Development / profiles helper."""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2002_12872_b200 as P  # noqa: E402
from paper_2002_12872_b200 import problems as pr  # noqa: E402

HBM = 6547.2  # GB/s, MEASURED_PEAKS.json

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1,c2,c2b,c3,c4,c4b")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--complex", action="store_true", help="complex coupling lambda(1 + 0.5i): the complex FP64 kernels")
a = ap.parse_args()
peak = P.fp64_peak_tflops(0)
for name in a.configs.split(","):
    t0 = time.time()
    p, o, desc = pr.config(name)
    cf = 4 if a.complex else 1  # complex: 4 real multiplies per product
    if a.complex:
        p = P.PartitionedProblem(p.d, p.delta, p.lam * (1 + 0.5j))
        desc += " complex"
    gen = time.time() - t0
    n = len(p.d)
    single = name.startswith("c4")
    dev = torch.device("cuda")
    d_t = torch.as_tensor(p.d, device=dev)
    if hasattr(p.delta, "rowptr"):
        delta_t = P.CsrMatrix(n, torch.as_tensor(p.delta.rowptr, device=dev),
                              torch.as_tensor(p.delta.cols, device=dev), torch.as_tensor(p.delta.vals, device=dev))
    else:
        delta_t = torch.as_tensor(p.delta, device=dev)
    pd = P.PartitionedProblem(d_t, delta_t, p.lam)
    plan = P.Plan(pd, single=single, row=n - 1)
    plan.begin()
    plan.steps(3)
    torch.cuda.synchronize()
    kms = plan.steps(a.steps, time_kernel=True) / a.steps
    s = torch.cuda.ExternalStream(P.default_context().stream_ptr)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    plan.steps(a.steps)
    e1.record(s)
    e1.synchronize()
    sms = e0.elapsed_time(e1) / a.steps
    plan.close()
    rec = {"config": name, "n": n, "desc": desc, "kernel_ms": kms, "step_ms": sms, "gen_s": round(gen, 2)}
    if single:
        nnz = p.delta.nnz
        byts = (12 + 8 * a.complex) * nnz + 8 * (n + 1) + 24 * n * (1 + a.complex)
        rec.update(bytes=byts, gbs=byts / (kms * 1e-3) / 1e9, hbm_frac=byts / (kms * 1e-3) / 1e9 / HBM)
    elif hasattr(p.delta, "rowptr"):
        nnz = p.delta.nnz
        byts = 16 * n * n * (1 + a.complex) + (12 + 8 * a.complex) * nnz + 8 * (n + 1) + 8 * n
        rec.update(bytes=byts, gbs=byts / (kms * 1e-3) / 1e9, hbm_frac=byts / (kms * 1e-3) / 1e9 / HBM,
                   tflops=2 * cf * nnz * n / (kms * 1e-3) / 1e12)
    else:
        rec.update(tflops=2 * cf * n ** 3 / (kms * 1e-3) / 1e12, fp64_frac=2 * cf * n ** 3 / (kms * 1e-3) / 1e12 / peak)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = P.dominant_eigenpair(pd, P.IterationOptions(**o)) if single else P.iterate_full(pd, P.IterationOptions(**o))
    torch.cuda.synchronize()
    rec.update(status=P.to_string(r.status), iterations=r.iterations, solve_ms=(time.perf_counter() - t0) * 1e3,
               solve_device_ms=r.device_ms)
    print(json.dumps(rec), flush=True)
print(json.dumps({"fp64_peak_tflops": peak}))
