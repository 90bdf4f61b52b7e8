"""CPU: the C-ABI library and the host-side logic, no GPU needed.

- libdpt_b200.so loads on a CPU-only host and exports every entry point that
  include/dpt_b200.h declares; without a device it fails loudly (no fallback).
- the O(n log n) degeneracy scan returns the reference's first (i, j).
- the device decision function (dpt_state.h, exposed as dpt_sm_decide_host),
  driven by a CPU model of the launch pipeline (tests/launch_sim.py), reproduces
  the reference's status / iteration count / read-offs.
- the sharded (multi-GPU) host logic: 2 gloo ranks, each owning half the rows,
  max-allreduce of the statistics and a final gather, equal to the unsharded run.
"""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2002_12872_b200 as P
import paper_2002_12872_b200._native as N
from oracle.bind import Checker
from paper_2002_12872_b200 import problems as pr
from paper_2002_12872_b200.dpt import PartitionedProblem

from conftest import has_gpu
from helpers import full_fixtures, load_full
from launch_sim import simulate

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
O = Checker("oracle")


def header_functions():
    src = open(os.path.join(ROOT, "include", "dpt_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dpt_[a-z0-9_]+)\s*\(", src)) - {"dpt_trace_fn"})


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(N.LIB_PATH)
    names = header_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert L.dpt_abi_version() == 2


def test_options_defaults_and_status_strings():
    o = N.dpt_options()
    N.lib().dpt_options_default(ctypes.byref(o))
    assert (o.tol, o.residual_tol, o.max_iter, o.divergence_threshold, o.cycle_window, o.degeneracy_tol) == \
        (1e-12, 1e-10, 10000, 1e8, 16, 1e-12)  # dpt.hpp:22-31
    assert [P.to_string(s) for s in P.ConvergenceStatus] == \
        ["Converged", "BoundedNonConverged", "Diverged", "MaxIterations"]


@pytest.mark.skipif(has_gpu(), reason="checks the no-device behaviour")
def test_no_cpu_fallback():
    with pytest.raises(P.NoDeviceError):
        P.iterate_full(pr.two_by_two(0.3))


def test_shape_errors_and_complex_marshalling():
    with pytest.raises(P.ShapeError):
        P.dpt._Marshal(PartitionedProblem(np.zeros(3), np.zeros((2, 2)), 0.1))
    m = P.dpt._Marshal(PartitionedProblem(np.zeros(2), np.zeros((2, 2)), 0.1 + 0.2j))
    assert m.prob.is_complex == 1 and m.prob.lambda_im == 0.2 and m.cplx
    # complex dtype with zero imaginary parts takes the real kernels, returns complex
    m = P.dpt._Marshal(PartitionedProblem(np.zeros(2, complex), np.zeros((2, 2), complex), 0.1 + 0j))
    assert m.prob.is_complex == 0 and m.cdtype and not m.cplx
    assert m.result(np.zeros(2)).dtype == np.complex128


def test_degeneracy_scan_matches_brute_force():
    rng = np.random.default_rng(3)
    for trial in range(300):
        n = int(rng.integers(1, 40))
        kind = trial % 4
        if kind == 0:
            d = rng.integers(0, max(n // 2, 1), size=n).astype(float)
        elif kind == 1:
            d = np.sort(rng.uniform(0, 1, n))
            if n > 3:
                d[n // 2] = d[n // 3] + 1e-13
        elif kind == 2:
            d = rng.uniform(-1e5, 1e5, n)
            if n > 2:
                d[-1] = d[1] + 5e-8
        else:
            d = np.arange(n, dtype=float)
        assert P.check_degenerate(d) == O.check_degenerate(d), d
    # threshold scales with the spread (test_partition.cpp:111-122)
    assert P.check_degenerate(np.array([1e5, 1e5 + 1e-9])) is None
    assert P.check_degenerate(np.array([0.0, 1e5, 1e5 + 1e-9])) == (1, 2)
    assert P.check_degenerate(np.array([0.0, 1e-16, 2.0])) == (0, 1)
    assert P.effective_window(16, 1024) == 3 and P.effective_window(16, 2000) == 0
    assert P.spectral_spread(np.array([3.0, -1.0, 2.0])) == 4.0


@pytest.mark.parametrize("path", full_fixtures(), ids=lambda p: p.split("/")[-1])
def test_decision_function_reproduces_reference(path):
    p, opts, z = load_full(path)
    q, a, eps, res = simulate(p, opts)
    assert q["status"] == int(z["status"])
    assert q["iterations"] == int(z["iterations"])
    if int(z["status"]) != 2:
        assert np.max(np.abs(a - z["a"])) < 1e-9
        assert np.max(np.abs(eps - z["eig"]) / np.maximum(1, np.abs(z["eig"]))) < 1e-10
    else:
        assert np.all(np.isnan(eps))


@pytest.mark.parametrize("lam,opts,want", [
    (0.0, {}, (0, 1)), (2.0, {}, (2, None)), (0.88, {}, (1, None)),
    (0.88, {"cycle_window": 0, "max_iter": 500}, (3, 500)), (0.3, {"max_iter": 3}, (3, 3)),
    (0.3, {"residual_tol": 0.0, "max_iter": 300}, (3, 300))])
def test_decision_function_known_answers(lam, opts, want):  # test_dpt.cpp:92-140
    p = pr.two_by_two(lam)
    q, a, eps, res = simulate(p, opts)
    r = O.iterate_full(p, opts)
    assert q["status"] == want[0] == r.status
    assert q["iterations"] == r.iterations and (want[1] is None or q["iterations"] == want[1])


def _sharded_worker(rank, world, port, path, outq):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p, opts, z = load_full(path)
    n = len(p.d)
    per = (n + world - 1) // world
    r0, r1 = min(n, rank * per), min(n, (rank + 1) * per)

    def allreduce(vec):
        t = torch.tensor(vec)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.numpy()

    q, a, eps, res = simulate(p, opts, allreduce=allreduce, shard=(r0, r1))
    pad = np.full((per, n), np.nan)
    pad[: r1 - r0] = a
    parts = [torch.zeros(per, n, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, torch.tensor(pad))
    ep = np.full(per, np.nan)
    ep[: r1 - r0] = eps
    eparts = [torch.zeros(per, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(eparts, torch.tensor(ep))
    if rank == 0:
        full = torch.cat(parts).numpy()[:n]
        eig = torch.cat(eparts).numpy()[:n]
        outq.put((q, full, eig))
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["full_c1_n48.npz", "full_c2_n64.npz", "full_c3_n96.npz",
                                  "full_two_by_two_lam0.88.npz"])
def test_sharded_two_ranks_gloo(name):
    """The multi-GPU decomposition (rows sharded, stats max-allreduced, final
    gather) on 2 CPU ranks equals the reference's unsharded result."""
    import socket

    import torch.multiprocessing as mp
    path = os.path.join(ROOT, "tests", "golden", name)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, path, q)) for r in range(2)]
    for pr_ in procs:
        pr_.start()
    res = q.get(timeout=240)
    for pr_ in procs:
        pr_.join(timeout=60)
    st, full, eig = res
    z = np.load(path)
    assert st["status"] == int(z["status"]) and st["iterations"] == int(z["iterations"])
    if int(z["status"]) != 2:
        assert np.max(np.abs(full - z["a"])) < 1e-9
        assert np.max(np.abs(eig - z["eig"]) / np.maximum(1, np.abs(z["eig"]))) < 1e-10


def test_library_needs_no_linear_algebra_libraries():
    """Row f2 runs on the repo's own kernels: libdpt_b200.so links neither
    cuBLAS nor cuSOLVER (the homotopy's GEMM / LU are csrc/linalg.cu)."""
    import subprocess
    so = os.path.join(ROOT, "paper_2002_12872_b200", "libdpt_b200.so")
    out = subprocess.run(["readelf", "-d", so], capture_output=True, text=True, check=True).stdout
    needed = [ln for ln in out.splitlines() if "NEEDED" in ln]
    assert needed and not any("cublas" in ln or "cusolver" in ln for ln in needed), needed
