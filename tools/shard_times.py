"""Per-rank step time of the sharded dense solve, emulated on one GPU
(DPT_SHARD_EMULATE=r/w: rank r's row shard, no communicator).  Development /
profiles helper: python tools/shard_times.py [worlds] (env DPT_DENSE_VARCOLS)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r"""
import sys, json
sys.path.insert(0, ".")
import paper_2002_12872_b200 as P
from paper_2002_12872_b200 import problems as pr
p, o, _ = pr.config("c2")
plan = P.Plan(p)
plan.begin(); plan.steps(3)
k = 20
kms = plan.steps(k, time_kernel=True) / k
print(json.dumps({"kernel_ms": kms}))
"""
worlds = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,8").split(",")]
for w in worlds:
    env = dict(os.environ, DPT_SHARD_EMULATE=f"0/{w}")
    out = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True)
    rec = json.loads(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else {"error": out.stderr[-300:]}
    rec.update(world=w, varcols=os.environ.get("DPT_DENSE_VARCOLS", "auto"))
    if "kernel_ms" in rec:
        rows = -(-4096 // w)
        rec["tflops"] = 2.0 * rows * 4096 * 4096 / (rec["kernel_ms"] * 1e-3) / 1e12
    print(json.dumps(rec))
