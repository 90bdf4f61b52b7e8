"""Profiling driver: a few fixed steps of one config through a Plan (used under ncu)."""
import argparse
import sys

sys.path.insert(0, ".")
import paper_2002_12872_b200 as P  # noqa: E402
from paper_2002_12872_b200 import problems as pr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--steps", type=int, default=4)
a = ap.parse_args()
p, o, desc = pr.config(a.config, a.n)
single = a.config.startswith("c4")
plan = P.Plan(p, single=single, row=len(p.d) - 1)
plan.begin()
plan.steps(a.steps)
print(desc, plan.stats())
