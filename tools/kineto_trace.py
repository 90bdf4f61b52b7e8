"""In-situ kernel timeline of one solve (torch.profiler / CUPTI activity
records: no cache flush, no serialisation, unlike an ncu launch list).
Prints per-kernel totals and the idle time between consecutive kernels."""
import argparse
import collections
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2002_12872_b200 as P  # noqa: E402
from paper_2002_12872_b200 import problems as pr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--cycle-window", type=int, default=None)
ap.add_argument("--json", default=None)
a = ap.parse_args()
p, o, desc = pr.config(a.config)
if a.cycle_window is not None:
    o = dict(o, cycle_window=a.cycle_window)
dev = torch.device("cuda")
if hasattr(p.delta, "rowptr"):
    delta = P.CsrMatrix(len(p.d), torch.as_tensor(p.delta.rowptr, device=dev), torch.as_tensor(p.delta.cols, device=dev),
                        torch.as_tensor(p.delta.vals, device=dev))
else:
    delta = torch.as_tensor(p.delta, device=dev)
pd = P.PartitionedProblem(torch.as_tensor(p.d, device=dev), delta, p.lam)
single = a.config.startswith("c4")
run = (lambda: P.dominant_eigenpair(pd, P.IterationOptions(**o))) if single else \
    (lambda: P.iterate_full(pd, P.IterationOptions(**o)))
run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r = run()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "Memcpy" not in e.name
      and "Memset" not in e.name]
ev.sort(key=lambda e: e.time_range.start)
tot = collections.OrderedDict()
for e in ev:
    k = e.name.split("(")[0][:60]
    c, t = tot.get(k, (0, 0.0))
    tot[k] = (c + 1, t + e.time_range.elapsed_us())
span = ev[-1].time_range.end - ev[0].time_range.start
busy = sum(e.time_range.elapsed_us() for e in ev)
print(desc, P.to_string(r.status), r.iterations, "device_ms", round(r.device_ms, 3))
for k, (c, t) in tot.items():
    print(f"  {k:60s} n={c:4d} total_us={t:10.1f} avg_us={t / c:8.2f}")
gaps = sorted(((ev[i + 1].time_range.start - ev[i].time_range.end), i) for i in range(len(ev) - 1))
if gaps:
    import statistics
    print("  gaps: median_us=%.2f max:" % statistics.median(g for g, _ in gaps),
          [(round(g, 1), ev[i].name.split("(")[0][-24:], ev[i + 1].name.split("(")[0][-24:]) for g, i in gaps[-4:]])
print(f"  span_us={span:.1f} busy_us={busy:.1f} idle_us={span - busy:.1f} per_iter_us={span / max(r.iterations, 1):.1f}")
if a.json:
    json.dump({"config": a.config, "kernels": {k: {"n": c, "total_us": t} for k, (c, t) in tot.items()},
               "span_us": span, "busy_us": busy, "iterations": r.iterations}, open(a.json, "w"), indent=1)
