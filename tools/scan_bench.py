"""Batched scan_domain throughput (cells/s) vs the reference's threaded
scan_domain on the host (dev helper; row f4)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2002_12872_b200 as P  # noqa: E402
from oracle.bind import ComplexReference  # noqa: E402
from paper_2002_12872_b200 import problems as pr  # noqa: E402
from paper_2002_12872_b200.dpt import IterationOptions, PartitionedProblem, ScanGrid, ScanMode  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--res", type=int, default=512)
ap.add_argument("--ref-res", type=int, default=64)
a = ap.parse_args()
R = ComplexReference()
threads = os.cpu_count() or 1
cases = [("two_by_two", pr.two_by_two(1.0), "Full", 0, ScanGrid(-1.2, 1.2, -1.0, 1.0)),
         ("random_uniform n=6", PartitionedProblem(*pr.random_uniform(6, 3), 0.0), "Full", 0,
          ScanGrid(-0.4, 0.4, -0.3, 0.3)),
         ("random_uniform n=16", PartitionedProblem(*pr.random_uniform(16, 3), 0.0), "Full", 0,
          ScanGrid(-0.2, 0.2, -0.2, 0.2)),
         ("oscillator n=64 row", PartitionedProblem(*pr.oscillator(64), 0.0), "SingleRow", 63,
          ScanGrid(0.0, 0.8, -0.3, 0.3))]
for name, p, mode, row, g in cases:
    o = IterationOptions(max_iter=300)
    grid = ScanGrid(g.re_min, g.re_max, g.im_min, g.im_max, a.res, a.res)
    P.scan_domain(p, ScanGrid(g.re_min, g.re_max, g.im_min, g.im_max, 8, 8), ScanMode(mode, row), o)
    t0 = time.perf_counter()
    out = P.scan_domain(p, grid, ScanMode(mode, row), o)
    tg = time.perf_counter() - t0
    rgrid = ScanGrid(g.re_min, g.re_max, g.im_min, g.im_max, a.ref_res, a.ref_res)
    t0 = time.perf_counter()
    rc, cls, its, _ = R.scan_domain(p, rgrid, mode, row, 0.0, {"max_iter": 300}, threads=threads)
    tr = time.perf_counter() - t0
    print(json.dumps({"case": name, "mode": mode, "gpu_cells": a.res * a.res, "gpu_s": round(tg, 5),
                      "gpu_cells_per_s": a.res * a.res / tg, "ref_cells": a.ref_res ** 2, "ref_threads": threads,
                      "ref_s": round(tr, 4), "ref_cells_per_s": a.ref_res ** 2 / tr,
                      "speedup": (a.res * a.res / tg) / (a.ref_res ** 2 / tr),
                      "mean_iterations": float(out.iterations.mean()),
                      "classes": [int((out.classes == c).sum()) for c in range(3)]}), flush=True)
