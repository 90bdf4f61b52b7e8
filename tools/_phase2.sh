cat > /tmp/ph.py <<'PY'
import sys; sys.path.insert(0, ".")
import paper_2002_12872_b200 as P
from paper_2002_12872_b200 import problems as pr
import time
for name in ["c4", "c3"]:
    p, o, _ = pr.config(name)
    f = (lambda: P.dominant_eigenpair(p, P.IterationOptions(**o))) if name == "c4" else (lambda: P.iterate_full(p, P.IterationOptions(**o)))
    f(); f()
    print("----", name, file=sys.stderr, flush=True)
    t0 = time.perf_counter(); f(); print(name, "wall ms", (time.perf_counter() - t0) * 1e3, file=sys.stderr, flush=True)
PY
for t in 4 8 12 16; do echo "threads $t"; DPT_COPY_THREADS=$t DPT_TIMING=1 timeout 300 python /tmp/ph.py 2>&1 | grep -E "staged|wall|upload|outputs" | tail -9; done > gpurun_out/phase2.txt 2>&1
