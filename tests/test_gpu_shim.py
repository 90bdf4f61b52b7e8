"""GPU: the drop-in boundary.  tests/cpp/drive.cpp is written against the
reference's public headers and calls every dpt.hpp entry point plus the
reference's own callers (compare_orders / truncation_agreement from
src/rspt.cpp, threaded scan_domain and bifurcation_scan from src/analysis.cpp),
unchanged.  Linked with the reference's src/dpt.cpp it is the CPU oracle
(build/drive_ref); linked with the shim + libdpt_b200.so it runs on the GPU
(build/drive_b200).  The two outputs must agree."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "build", "drive_ref")
B200 = os.path.join(ROOT, "build", "drive_b200")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (os.path.exists(REF) and os.path.exists(B200)),
                                 reason="build/drive_* not built (needs /root/reference at build time)")]


def run(path):
    out = subprocess.run([path], capture_output=True, text=True, timeout=900, check=True).stdout
    d = {}
    for line in out.splitlines():
        k, v = line.split(" ", 1)
        d[k] = v
    return d


def test_shim_matches_reference_callers():
    ref, got = run(REF), run(B200)
    assert ref.keys() == got.keys()
    for k, rv in ref.items():
        gv = got[k]
        if k.endswith(".status") or k == "done":
            assert gv == rv, k
            continue
        r, g = float(rv), float(gv)
        if k.endswith("iterations") or k.startswith("compare.k_") or ".iters[" in k:
            assert abs(r - g) <= 1, (k, r, g)
        elif k.startswith("scan_") or k.endswith("converged"):
            assert r == g, (k, r, g)
        else:
            assert abs(r - g) <= 1e-9 * max(1.0, abs(r)), (k, r, g)
