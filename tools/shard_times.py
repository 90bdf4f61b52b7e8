"""Per-rank step time of the sharded dense solve, emulated on one GPU
(DPT_SHARD_EMULATE=r/w: rank r's row shard, no communicator).  Development /
profiles helper:  python tools/shard_times.py [--config c2|c5] [--worlds 1,2,4,8]
Rank 0 holds the largest shard (ceil(n / w) rows), so its time is the step's."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_12872_b200 as P  # noqa: E402
from paper_2002_12872_b200 import problems as pr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--worlds", default="1,2,4,8")
ap.add_argument("--steps", type=int, default=0)
a = ap.parse_args()
p, o, _ = pr.config(a.config)
n = len(p.d)
k = a.steps or (20 if n <= 8192 else 2)
peak = P.fp64_peak_tflops(0)
for w in [int(x) for x in a.worlds.split(",")]:
    os.environ["DPT_SHARD_EMULATE"] = f"0/{w}"
    plan = P.Plan(p)
    plan.begin()
    plan.steps(1 if n > 8192 else 3)
    kms = plan.steps(k, time_kernel=True) / k
    plan.close()
    rows = -(-n // w)
    tf = 2.0 * rows * n * n / (kms * 1e-3) / 1e12
    print(json.dumps({"config": a.config, "n": n, "world": w, "rows_rank0": rows, "kernel_ms": kms, "tflops": tf,
                      "fp64_frac": tf / peak}), flush=True)
os.environ.pop("DPT_SHARD_EMULATE", None)
