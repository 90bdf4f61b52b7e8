"""Matrix Market ingestion throughput (row f3): the library's threaded reader
vs the reference's read_matrix_market on a c4-shaped file (dev helper)."""
import argparse
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2002_12872_b200 as P  # noqa: E402
from oracle.bind import ReferenceMatrixMarket  # noqa: E402
from paper_2002_12872_b200 import problems as pr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--threads", type=int, default=0)
ap.add_argument("--ref", type=int, default=1)
a = ap.parse_args()
csr = pr.csr_fixed_per_row(a.n, 3, 16)
d = tempfile.mkdtemp()
path = os.path.join(d, "delta.mtx")
t0 = time.perf_counter()
P.write_matrix_market(csr, path, threads=a.threads)
tw = time.perf_counter() - t0
size = os.path.getsize(path)
t0 = time.perf_counter()
m = P.read_matrix_market(path, threads=a.threads)
tr = time.perf_counter() - t0
assert np.array_equal(m.rowptr, csr.rowptr) and np.array_equal(m.cols, csr.cols)
assert np.array_equal(m.vals.view(np.int64), csr.vals.view(np.int64))
rec = {"n": a.n, "nnz": int(csr.nnz), "file_mb": size / 1e6, "threads": a.threads or os.cpu_count(),
       "write_s": tw, "read_s": tr, "read_mb_s": size / 1e6 / tr, "read_entries_per_s": csr.nnz / tr}
if a.ref:
    R = ReferenceMatrixMarket()
    t0 = time.perf_counter()
    rc, msg, ref = R.read(path)
    rec["ref_read_s"] = time.perf_counter() - t0
    rec["speedup"] = rec["ref_read_s"] / tr
    assert rc == 0 and np.array_equal(ref[1], csr.rowptr)
print(json.dumps(rec))
os.remove(path)
