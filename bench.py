#!/usr/bin/env python
"""bench.py -- DPT iteration throughput on B200 (BASELINE.json metric).

Workloads (SURVEY.md §8(d) recipe, synthetic, seeded):
  N = 1 (default): BASELINE.json configs[1] -- dense unsymmetric full
          diagonalisation, n = 4096, FP64, seed 1, lambda = 0.5/sqrt(n).  Under
          reference semantics it terminates Diverged at k = 4, so, as BASELINE.md
          prescribes, throughput is timed over a fixed number of map applications
          (iterate_fixed semantics, dpt.hpp:94-96).
  N > 1:  BASELINE.json configs[4] -- dense symmetric n = 32768, seed 4, the
          north_star's column-sharded multi-GPU config: rows of A (the paper's
          columns) sharded over the ranks, Delta replicated, one NCCL
          max-allreduce of the step statistics per iteration, final allgather.
          (--workload c2|c5 overrides the choice.)
One STEP = one DPT iteration = one fused K1 launch (P = A Delta^T GEMM + map +
residual + step-norm epilogue) + the fold (+ allreduce + decision) kernels.
Metric unit: iterations / s (whole job: every rank advances the same iteration).

  value   device-resident: inputs in HBM, CUDA events on the solver's stream
          around exactly K steps, max over ranks.
  e2e     the public API a user calls (paper_2002_12872_b200.iterate_full) on
          pinned host arrays: H2D of theta + Delta, the solve to its terminal
          status, D2H of A / eigenvalues / residuals; iterations / wall second.
  roofline  the dense step kernel alone (events around each launch): 2 n^2 rows
          FLOP per launch / average launch time, against the FP64 tensor-core
          peak measured in this run (DMMA probe; MEASURED_PEAKS.json has no FP64).
  cpu_baseline  the reference's own implementation (oracle/_ref, compiled from
          /root/reference/proj/src) on a bounded row sample, all host threads.
  time_to_converge  (N = 1) the public iterate_full call, device-resident
          inputs, to the terminal status: c2 (Diverged 4) and its converging
          companion c2b (theta_i = i).

--gpus N without torchrun re-launches itself under torch.distributed.run with
N ranks (and fails if fewer than N GPUs are visible).
--impl reference times only the reference arm (rank 0; other ranks exit 0).
--baselines prints the per-config reference-vs-B200 table.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="auto", choices=["auto", "c2", "c5"],
                    help="auto: c2 (configs[1]) at N = 1, c5 (configs[4]) at N > 1")
    ap.add_argument("--size", type=int, default=0, help="override n (testing only)")
    ap.add_argument("--e2e-calls", type=int, default=0, help="public calls timed for e2e (0: 5 for c2, 1 for c5)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--baselines", action="store_true",
                    help="instead of the bench line: the reference's own CPU solver on every BASELINE config "
                         "(time to its terminal status, one core) next to the B200 public call, plus the "
                         "lambda-plane scan and Matrix Market legs (several minutes)")
    return ap.parse_args()


WORKLOADS = {
    "c2": ("BASELINE configs[1]: dense unsymmetric DPT full diagonalisation, n={n}, FP64, seed 1, "
           "theta ~ sorted U(0,n) with adjacent gaps >= 1e-3, Delta N(0,1) off-diagonal, "
           "lambda=0.5/sqrt(n); step = one map application (iterate_fixed semantics)", 4096),
    "c5": ("BASELINE configs[4]: dense symmetric DPT full diagonalisation, n={n}, FP64, seed 4, theta_i = i, "
           "Delta symmetrised N(0,1) with zero diagonal, lambda=0.5/sqrt(n), tol 1e-12; rows of A column-"
           "sharded over the ranks, Delta replicated; step = one map application (iterate_fixed semantics)", 32768),
}


def pick_workload(args, world):
    wl = args.workload if args.workload != "auto" else ("c2" if world == 1 else "c5")
    return wl, (args.size or WORKLOADS[wl][1])


def workload_config(wl, n, world):
    return {
        "workload": WORKLOADS[wl][0].format(n=n),
        "n": n,
        "lambda": 0.5 / math.sqrt(n),
        "flop_per_step": 2.0 * n ** 3,
        "l2": f"inputs larger than L2: A_k {n * n * 8 / 2**20 / world:.0f} MiB per rank + Delta "
              f"{n * n * 8 / 2**20:.0f} MiB per step vs 126 MB L2 (no flush needed)",
        "parallelism": f"rows of A sharded over {world} rank(s) (dp{world}), Delta replicated, NCCL max-allreduce "
                       "per iteration" if world > 1 else "single GPU",
    }


def make_inputs(wl, n, pinned=False):
    from paper_2002_12872_b200 import problems as pr
    p, o, desc = pr.config(wl, n)
    if pinned:
        import torch
        d = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
        a = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy()
        d[:] = p.d
        a[:] = p.delta
        p.d, p.delta = d, a
    return p, o


# ------------------------------------------------------------------ clocks ----
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------- reference arm ----
def reference_sample(p, a_rows_src, threads, rows_per_thread, lam):
    """Times the reference's own step (matmul with delta_t + map, proj/src/
    matrix.cpp:130-143, dpt.cpp:136-144) on threads x rows_per_thread rows.
    Returns (wall seconds, rows)."""
    from oracle.bind import Checker
    import ctypes
    R = Checker("reference")
    pr, keep = R._prob(p)
    h = R.L.ref_prepare(ctypes.byref(pr))
    try:
        rows = threads * rows_per_thread
        a = np.ascontiguousarray(a_rows_src[:rows])
        out = np.empty_like(a)
        n = p.d.shape[0]

        def work(t):
            r0 = t * rows_per_thread
            R.L.ref_prepared_step_rows(h, r0, rows_per_thread, a[r0:].ctypes.data, lam, out[r0:].ctypes.data)

        ths = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
        t0 = time.perf_counter()
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        return time.perf_counter() - t0, rows, out
    finally:
        R.L.ref_release(h)


def first_iterate_rows(p, rows):
    """Dense rows of A_1 = F(I) (the reference's matmul zero-skips I, so a dense
    iterate is needed for a representative sample): A_1(i,j) = lam theta(i,j) Delta(j,i)."""
    d, D, lam = p.d, p.delta, p.lam
    out = np.empty((rows, d.shape[0]))
    for i in range(rows):
        with np.errstate(divide="ignore"):
            g = 1.0 / (d[i] - d)
        g[i] = 0.0
        out[i] = (lam * g) * D[:, i]
        out[i, i] = 1.0
    return out


def reference_inputs(wl, n):
    """The reference arm's inputs, built by oracle/gen.py (numpy restatement of
    the same recipe) so the arm maps none of this repo's shared libraries."""
    from types import SimpleNamespace
    from oracle import gen
    d, delta, lam = gen.dense_config(wl, n)
    return SimpleNamespace(d=d, delta=delta, lam=lam)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(max(args.gpus, 1))))
    if rank != 0:
        return 0
    from oracle.bind import available
    wl, n = pick_workload(args, world)
    cfg = workload_config(wl, n, world)
    if not available("reference"):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libdynspec_ref.so not built"}))
        return 0
    p = reference_inputs(wl, n)
    threads = os.cpu_count() or 1
    rpt = 4 if wl == "c2" else 1  # c5: one reference row is n^2 = 1.1e9 complex MACs (~4 s)
    a_rows = first_iterate_rows(p, threads * rpt)
    for _ in range(max(min(args.warmup, 1), 0)):
        reference_sample(p, a_rows, threads, rpt, p.lam)
    secs = []
    for _ in range(args.steps if wl == "c2" else min(args.steps, 2)):
        s, rows, _ = reference_sample(p, a_rows, threads, rpt, p.lam)
        secs.append(s)
    t = float(np.mean(secs))
    rows = threads * rpt
    it_s = (rows / n) / t
    sample = (f"{rows} of {n} rows of one {wl} iteration per step (reference matmul(A_rows, delta_t) "
              f"+ map, complex<double> as in the reference), {threads} threads x {rpt} rows; "
              f"iterations/s = sampled fraction / wall time (time per iteration extrapolated x{n / rows:.1f}); "
              "inputs from oracle/gen.py")
    print(json.dumps({
        "impl": "reference", "metric": metric_name(n), "value": it_s,
        "unit": "iter/s", "n_gpus": 0, "steps": len(secs), "warmup": args.warmup,
        # a step of this arm is the timed row sample (so steps x ms_per_step is the
        # timed wall time); the full iteration it stands for is extrapolated
        "ms_per_step": t * 1e3, "ms_per_full_iteration_extrapolated": 1e3 / it_s, "higher_is_better": True, "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None, "dtype": "f64 (complex<double>)", "data": "synthetic", "config": cfg,
        "sample_rows": rows, "extrapolation_factor": n / rows, "sample_wall_s_per_step": t,
        "cpu_baseline": {"value": it_s, "unit": "iter/s", "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": it_s, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


def metric_name(n):
    return f"DPT iterations/s (dense n={n} FP64 step)"


# ------------------------------------------------------ baselines table ----
def _timed(fn, reps=1):
    best, out = None, None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best, out


def run_baselines():
    """BASELINE.md §3's CPU baseline plan, measured on this box in one run: the
    reference's own solver (oracle/_ref, one core -- it is single-threaded) to
    its terminal status on c1 / c3 / c4 / c4b, one c2 iteration via
    iterate_fixed, against the B200 public call (host arrays in and out; warm,
    best of 3; and device-resident inputs).  Then the reference's threaded
    scan_domain vs the batched scan, and its Matrix Market reader vs ours."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    import torch
    import paper_2002_12872_b200 as P
    from oracle.bind import Checker, ComplexReference, ReferenceMatrixMarket, available
    from paper_2002_12872_b200 import problems as pr
    from paper_2002_12872_b200.dpt import CsrMatrix, IterationOptions, PartitionedProblem, ScanGrid, ScanMode
    if not available("reference"):
        print(json.dumps({"baselines": "unavailable", "why": "oracle/_ref not built"}))
        return 0
    R = Checker("reference")
    host = {"cpu": os.cpu_count(), "model": platform_cpu()}

    def dev_problem(p):
        dv = torch.device("cuda")
        d = torch.as_tensor(p.d, device=dv)
        if hasattr(p.delta, "rowptr"):
            delta = CsrMatrix(len(p.d), torch.as_tensor(p.delta.rowptr, device=dv),
                              torch.as_tensor(p.delta.cols, device=dv), torch.as_tensor(p.delta.vals, device=dv))
        else:
            delta = torch.as_tensor(p.delta, device=dv)
        return PartitionedProblem(d, delta, p.lam)

    for name in ("c1", "c4", "c4b", "c3"):
        p, o, desc = pr.config(name)
        single = name.startswith("c4")
        if single:
            tr, r = _timed(lambda: R.dominant_eigenpair(p, o))
            call = lambda q: P.dominant_eigenpair(q, IterationOptions(**o))  # noqa: E731
        else:
            tr, r = _timed(lambda: R.iterate_full(p, o))
            call = lambda q: P.iterate_full(q, IterationOptions(**o))  # noqa: E731
        tg, g = _timed(lambda: call(p), reps=3)
        pd = dev_problem(p)
        torch.cuda.synchronize()
        td, gd = _timed(lambda: call(pd), reps=3)
        print(json.dumps({"config": name, "workload": desc,
                          "reference": {"status": STATUS_NAMES[r.status], "iterations": r.iterations, "s": tr,
                                        "cores": 1, "host": host},
                          "b200": {"status": P.to_string(g.status), "iterations": g.iterations,
                                   "host_arrays_s": tg, "device_inputs_s": td},
                          "speedup_host_arrays": tr / tg}), flush=True)
    # c2: one reference iteration (a full c2 run is ~11 min on one core; it diverges at k = 4).
    # iterate_fixed(1) only needs P(I) (the reference's matmul skips I's zeros); k = 2 adds the
    # first full product, so the difference is one iteration.
    p, o, desc = pr.config("c2")
    t1, _ = _timed(lambda: R.iterate_fixed(p, 1, p.lam))
    t2, _ = _timed(lambda: R.iterate_fixed(p, 2, p.lam))
    tr = t2 - t1
    plan = P.Plan(p)
    plan.begin()
    plan.steps(3)
    torch.cuda.synchronize()
    t_step = plan.steps(20, time_kernel=True) / 20 * 1e-3
    plan.close()
    print(json.dumps({"config": "c2", "workload": desc + "; one iteration (reference: iterate_fixed k = 2 minus k = 1)",
                      "reference": {"s_per_iteration": tr, "cores": 1, "host": host},
                      "b200": {"s_per_iteration_kernel": t_step}, "speedup": tr / t_step}), flush=True)
    # lambda-plane scans (row f4): the reference's scan_domain on all host threads vs the batched kernel
    C = ComplexReference()
    threads = os.cpu_count() or 1
    cases = [("two_by_two", pr.two_by_two(1.0), "Full", 0, (-1.2, 1.2, -1.0, 1.0)),
             ("random_uniform n=16", PartitionedProblem(*pr.random_uniform(16, 3), 0.0), "Full", 0,
              (-0.2, 0.2, -0.2, 0.2)),
             ("oscillator n=64 row", PartitionedProblem(*pr.oscillator(64), 0.0), "SingleRow", 63, (0.0, 0.8, -0.3, 0.3))]
    for name, p, mode, row, g in cases:
        o = IterationOptions(max_iter=300)
        P.scan_domain(p, ScanGrid(*g, 8, 8), ScanMode(mode, row), o)
        tg = min(_timed(lambda: P.scan_domain(p, ScanGrid(*g, 512, 512), ScanMode(mode, row), o))[0]
                 for _ in range(3))  # best of 3: one 65 ms call right after the c2 legs once read 2.5x slow
        tr, _ = _timed(lambda: C.scan_domain(p, ScanGrid(*g, 64, 64), mode, row, 0.0, {"max_iter": 300},
                                              threads=threads))
        print(json.dumps({"scan": name, "mode": mode, "b200_cells_per_s": 512 * 512 / tg,
                          "reference_cells_per_s": 64 * 64 / tr, "reference_threads": threads,
                          "speedup": (512 * 512 / tg) / (64 * 64 / tr)}), flush=True)
    # Matrix Market (row f3): a c4-shaped file, the reference's reader vs ours
    import tempfile
    csr = pr.csr_fixed_per_row(1 << 20, 3, 16)
    path = os.path.join(tempfile.mkdtemp(), "delta.mtx")
    P.write_matrix_market(csr, path)
    tg, m = _timed(lambda: P.read_matrix_market(path))
    tr, (rc, _, ref) = _timed(lambda: ReferenceMatrixMarket().read(path))
    assert rc == 0 and np.array_equal(m.rowptr, ref[1]) and np.array_equal(m.cols, csr.cols)
    print(json.dumps({"matrix_market": "read c4-shaped file", "mb": os.path.getsize(path) / 1e6, "b200_lib_s": tg,
                      "reference_s": tr, "speedup": tr / tg}), flush=True)
    os.remove(path)
    return 0


STATUS_NAMES = ["Converged", "BoundedNonConverged", "Diverged", "MaxIterations"]


def platform_cpu():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------ B200 arm ----
def other_configs(P, torch, ctx, local, fp64_peak):
    """c1 / c3 / c4 / c4b next to the bench line: event-timed step kernel over
    20 fixed steps (c1 / c3: K1 / K2, c4: K3) with its roofline fraction (FP64
    against the DMMA peak for dense, algorithmic HBM bytes against
    MEASURED_PEAKS.json for CSR / row map), and the public call to the terminal
    status with device-resident inputs (best of 3)."""
    from paper_2002_12872_b200 import problems as pr
    hbm = 6551.0
    try:
        hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    dev = torch.device("cuda", local)
    out = {}
    for name in ("c1", "c3", "c4", "c4b"):
        p, o, desc = pr.config(name)
        n = len(p.d)
        if hasattr(p.delta, "rowptr"):
            delta = P.CsrMatrix(n, torch.as_tensor(p.delta.rowptr, device=dev), torch.as_tensor(p.delta.cols, device=dev),
                                torch.as_tensor(p.delta.vals, device=dev))
        else:
            delta = torch.as_tensor(p.delta, device=dev)
        pd = P.PartitionedProblem(torch.as_tensor(p.d, device=dev), delta, p.lam)
        single = name.startswith("c4")
        plan = P.Plan(pd, single=single, row=n - 1, ctx=ctx)
        plan.begin()
        plan.steps(3)
        kms = plan.steps(20, time_kernel=True) / 20
        plan.close()
        rec = {"workload": desc, "kernel_ms": kms}
        if single:
            byts = 12 * p.delta.nnz + 8 * (n + 1) + 24 * n
            rec.update(kernel="single_u16w_kernel (K3)", bound="hbm", gbs=byts / (kms * 1e-3) / 1e9,
                       frac=byts / (kms * 1e-3) / 1e9 / hbm, algorithmic_bytes=byts)
            # what binds it (K3): one random 32-byte sector per SM clock on the miss path to L2;
            # sectors per step = nnz gathers + the streamed bytes / 32
            sm, ghz = 148, 1.965
            sectors = p.delta.nnz + byts / 32.0
            floor_ms = sectors / sm / (ghz * 1e9) * 1e3
            rec.update(binding="SM miss path to L2 (one sector per SM clock)", sector_floor_ms=floor_ms,
                       frac_of_sector_floor=floor_ms / kms)
        elif hasattr(p.delta, "rowptr"):
            byts = 16 * n * n + 12 * p.delta.nnz + 8 * (n + 1) + 8 * n
            rec.update(kernel="csr_step_kernel (K2)", bound="hbm", gbs=byts / (kms * 1e-3) / 1e9,
                       frac=byts / (kms * 1e-3) / 1e9 / hbm, algorithmic_bytes=byts)
            # what binds it (K2): n * nnz random 8-byte shared-memory gathers through the
            # 128 B/clk L1 data pipe of each SM
            sm, ghz = 148, 1.965
            floor_ms = float(n) * p.delta.nnz * 8.0 / (sm * 128.0 * ghz * 1e9) * 1e3
            rec.update(binding="L1 data pipe (shared-memory gathers)", smem_gather_floor_ms=floor_ms,
                       frac_of_gather_floor=floor_ms / kms)
        else:
            tf = 2.0 * n ** 3 / (kms * 1e-3) / 1e12
            rec.update(kernel="dense_step_kernel (K1)", bound="tensor", tflops=tf, frac=tf / fp64_peak)
        call = (lambda: P.dominant_eigenpair(pd, P.IterationOptions(**o), ctx=ctx)) if single else \
            (lambda: P.iterate_full(pd, P.IterationOptions(**o), ctx=ctx))
        call()
        best, r = None, None
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = call()
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) * 1e3
            best = dt if best is None else min(best, dt)
        rec.update(status=P.to_string(r.status), iterations=r.iterations, solve_wall_ms=best,
                   solve_device_ms=r.device_ms)
        out[name] = rec
        del pd, delta
    out["how"] = ("kernel: CUDA events around each of 20 fixed steps on the solver stream; solve: public call, "
                  "device-resident inputs, warm, best of 3")
    return out


def spawn(args):
    """--gpus N outside torchrun: re-launch this script with N ranks (one per GPU)."""
    import socket
    if args.impl == "b200":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} requested but only {have} GPU(s) are visible", file=sys.stderr)
            return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # keep NCCL's init lines (nranks) visible
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.baselines:
        return run_baselines()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn(args)
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    import paper_2002_12872_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    if torch.cuda.device_count() < world:
        print(f"bench.py: {world} ranks but only {torch.cuda.device_count()} GPU(s) visible", file=sys.stderr)
        return 2
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl, n = pick_workload(args, world)
    e2e_calls = args.e2e_calls or (5 if wl == "c2" else 1)
    ctx = P.Context(local)
    if world > 1:
        uid = [P.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.set_comm(rank, world, uid[0])

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    t_gen = time.perf_counter()
    p, opts = make_inputs(wl, n)
    t_gen = time.perf_counter() - t_gen
    stream = torch.cuda.ExternalStream(ctx.stream_ptr)
    plan = P.Plan(p, ctx=ctx)
    plan.begin()
    plan.steps(max(args.warmup, 3))
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)  # let the sampler attach before the timed region
    launches0 = ctx.launches
    barrier()
    ev0.record(stream)
    plan.steps(args.steps)
    ev1.record(stream)
    ev1.synchronize()
    barrier()
    launches = ctx.launches - launches0
    ms_total = max_over_ranks(ev0.elapsed_time(ev1))
    clk = clocks.stop()
    ms_per_step = ms_total / args.steps
    value = 1e3 / ms_per_step  # whole-job iterations per second (all ranks advance the same iteration)

    # roofline: the dense step kernel alone, events on its own stream (max over ranks)
    kernel_steps = min(args.steps, 50 if wl == "c2" else 3)
    kms = max_over_ranks(plan.steps(kernel_steps, time_kernel=True) / kernel_steps)
    rows_local = (n + world - 1) // world
    flop_launch = 2.0 * rows_local * n * n
    achieved = flop_launch / (kms * 1e-3) / 1e12
    peak = P.fp64_peak_tflops(local)
    traffic, traffic_src = None, None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof) and wl == "c2" and world == 1:
        try:
            rec = json.load(open(prof)).get("latest:prof_dense_c2", {})
            traffic = rec.get("dram_bytes_per_launch")
            traffic_src = (f"ncu --set full capture {rec.get('capture')} of the same kernel at this workload "
                           f"(profiles/ncu_summary.json; dram__bytes_read.sum + dram__bytes_write.sum per launch, "
                           f"cold-cache replay) -- not measured inside this run") if traffic else None
        except Exception:
            traffic = None
    plan.close()

    # N > 1: the same workload's one-GPU step on rank 0 (the others wait), so the
    # line carries its own single-GPU point of the c5 scaling curve
    one_gpu = None
    if world > 1:
        if rank == 0:
            c1 = P.Context(local)
            pl1 = P.Plan(p, ctx=c1)
            pl1.begin()
            pl1.steps(1)
            k1 = min(args.steps, 3)
            ms1 = pl1.steps(k1, time_kernel=True) / k1
            s1 = torch.cuda.ExternalStream(c1.stream_ptr)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s1)
            pl1.steps(k1)
            e1.record(s1)
            e1.synchronize()
            step1 = e0.elapsed_time(e1) / k1
            pl1.close()
            c1.close()
            one_gpu = {"value": 1e3 / step1, "unit": "iter/s", "ms_per_step": step1, "k1_ms": ms1,
                       "how": "rank 0 alone, unsharded plan of the same problem, events on its stream"}
        barrier()

    # e2e: the public API on pinned host arrays, solve to the terminal status
    pe, oe = make_inputs(wl, n, pinned=True)
    io = P.IterationOptions(**oe)
    outs = (torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy(),
            torch.empty(n, dtype=torch.float64, pin_memory=True).numpy(),
            torch.empty(n, dtype=torch.float64, pin_memory=True).numpy())
    if wl == "c2":
        P.iterate_full(pe, io, ctx=ctx, out=outs)  # warm-up (first-call allocations)
    barrier()
    t0 = time.perf_counter()
    iters = 0
    for _ in range(e2e_calls):
        r = P.iterate_full(pe, io, ctx=ctx, out=outs)
        iters += r.iterations
    barrier()
    wall = max_over_ranks(time.perf_counter() - t0)
    e2e = {"value": iters / wall, "unit": "iter/s",
           "h2d_bytes_per_step": int((n * n + n) * 8 / max(r.iterations, 1)),
           "d2h_bytes_per_step": int((n * n + 2 * n) * 8 / max(r.iterations, 1)),
           "call": f"iterate_full({wl}) pinned host arrays in and out -> {P.to_string(r.status)} at "
                   f"k={r.iterations}, {wall / e2e_calls * 1e3:.2f} ms per call (upload, solve, download)"
                   + (f", {world} ranks (allgather of A to every rank)" if world > 1 else "")}
    del pe, outs

    # time to the terminal status through the public call, device-resident inputs
    ttc = None
    if world == 1 and wl == "c2":
        ttc = {}
        for name in ("c2", "c2b"):
            from paper_2002_12872_b200 import problems as pr
            q, oq, _ = pr.config(name, n)
            dv = torch.device("cuda", local)
            qd = P.PartitionedProblem(torch.as_tensor(q.d, device=dv), torch.as_tensor(q.delta, device=dv), q.lam)
            P.iterate_full(qd, P.IterationOptions(**oq), ctx=ctx)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rr = P.iterate_full(qd, P.IterationOptions(**oq), ctx=ctx)
            torch.cuda.synchronize()
            ttc[name] = {"status": P.to_string(rr.status), "iterations": rr.iterations,
                         "wall_ms": (time.perf_counter() - t0) * 1e3, "device_ms": rr.device_ms}
            del qd
        ttc["how"] = ("public iterate_full, device-resident theta/Delta, results on the device; warm call; "
                      "c2b = c2 with theta_i = i (the converging companion, SURVEY.md §8(d))")
    elif world > 1 or wl == "c5":
        ttc = {wl: {"status": P.to_string(r.status), "iterations": r.iterations,
                    "wall_ms_with_host_copies": wall / e2e_calls * 1e3}}

    # N = 1: the other BASELINE configs in the same run (kernel per step with its
    # roofline fraction, and time to the terminal status through the public call
    # with device-resident inputs), so the driver's record covers every config
    others = None
    if world == 1 and wl == "c2" and not args.size:
        others = other_configs(P, torch, ctx, local, peak)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle.bind import available
            if available("reference"):
                threads = os.cpu_count() or 1
                rpt = 8 if wl == "c2" else 1
                a_rows = first_iterate_rows(p, threads * rpt)
                s, rows, _ = reference_sample(p, a_rows, threads, rpt, p.lam)
                cpu = {"value": (rows / n) / s, "unit": "iter/s", "cores": threads, "kind": "reference",
                       "sample": f"{rows} of {n} rows of one {wl} iteration (reference matmul(A_rows, delta_t) + map, "
                                 f"complex<double>), {threads} threads; iter/s = fraction / wall "
                                 f"(extrapolated x{n / rows:.1f})"}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "iter/s", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": metric_name(n), "value": value, "unit": "iter/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (SURVEY.md §8(d) recipe, seeded)",
            "config": workload_config(wl, n, world),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "kernel": "dense_step_kernel (K1)", "kernel_ms": kms,
                         "flop_per_launch": flop_launch,
                         "peak_source": "FP64 DMMA probe measured in this run (MEASURED_PEAKS.json has no FP64 entry)"},
            "e2e": e2e, "time_to_converge": ttc, "cpu_baseline": cpu, "clocks": clk, "gpu_launches": int(launches),
            "other_configs": others,
            "tflops_per_step": 2.0 * n ** 3 / (ms_per_step * 1e-3) / 1e12,
            "input_gen_s": t_gen,
        }
        if world > 1:
            line["per_rank"] = {"k1_ms_max": kms, "step_ms": ms_per_step,
                                "fold_allreduce_decide_ms": ms_per_step - kms,
                                "rows_per_rank": rows_local}
            line["same_workload_1gpu"] = one_gpu
    # tear the communicators down BEFORE printing: with NCCL_DEBUG=INFO their
    # shutdown lines would otherwise follow the JSON line
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        sys.stdout.flush()
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
