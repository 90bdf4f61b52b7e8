"""GPU: K1's tile configurations and the stream-K variant agree to rounding.
Each P(i, j) sums over k in the same order in every one-tile configuration, but
the next iterate's diagonal d(i) = sum_j A'(i, j) Delta(i, j) is folded from
per-tile partial sums whose grouping follows the tile width (128 vs 64), and
stream-K adds a tile's k-range parts at the end -- so iterates agree to a few
ulps, and statuses / iteration counts agree."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2002_12872_b200 as P
from paper_2002_12872_b200 import problems as pr
from paper_2002_12872_b200.dpt import PartitionedProblem
name, n, cplx = sys.argv[1], int(sys.argv[2]), sys.argv[3] == "1"
p, o, _ = pr.config(name, n)
if cplx:
    p = PartitionedProblem(p.d, p.delta, p.lam * (1 + 0.5j))
a = P.iterate_fixed(p, 3, p.lam)
r = P.iterate_full(p, P.IterationOptions(**o))
np.savez(sys.argv[4], a=a, eig=r.eigenvalues, status=int(r.status), iterations=r.iterations)
"""


def run(tmp_path, tag, env, *args):
    f = str(tmp_path / f"{tag}.npz")
    subprocess.run([sys.executable, "-c", SCRIPT, *args, f], cwd=ROOT, env=dict(os.environ, **env), check=True,
                   timeout=600)
    return np.load(f)


def test_big_tile_configurations_agree(tmp_path):
    a = run(tmp_path, "cfg1", {"DPT_DENSE_CFG": "1"}, "c2b", "2048", "0")
    b = run(tmp_path, "cfg2", {"DPT_DENSE_CFG": "2"}, "c2b", "2048", "0")
    assert np.max(np.abs(a["a"] - b["a"])) < 1e-12
    assert int(a["status"]) == int(b["status"]) and int(a["iterations"]) == int(b["iterations"])
    assert np.max(np.abs(a["eig"] - b["eig"]) / np.maximum(1.0, np.abs(b["eig"]))) < 1e-12


def test_stream_k_matches_one_tile(tmp_path):
    sk = run(tmp_path, "sk", {"DPT_DENSE_SK": "1"}, "c1", "1024", "1")
    one = run(tmp_path, "one", {"DPT_DENSE_SK": "0"}, "c1", "1024", "1")
    assert int(sk["status"]) == int(one["status"]) and abs(int(sk["iterations"]) - int(one["iterations"])) <= 1
    assert np.max(np.abs(sk["a"] - one["a"])) < 1e-10
    if int(sk["iterations"]) == int(one["iterations"]):
        assert np.max(np.abs(sk["eig"] - one["eig"]) / np.maximum(1.0, np.abs(one["eig"]))) < 1e-12
