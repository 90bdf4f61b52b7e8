timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -3
cat > /tmp/h.py <<'PY'
import sys, time
sys.path.insert(0, ".")
import paper_2002_12872_b200 as P
from paper_2002_12872_b200 import problems as pr
p, o, _ = pr.config("c1", 1024)
P.homotopy_solve(p, 2, P.IterationOptions(**o))
t0 = time.perf_counter(); h = P.homotopy_solve(p, 2, P.IterationOptions(**o)); t1 = time.perf_counter()
print("homotopy c1 n=1024 stages=2:", P.to_string(h.status), h.iterations, "wall_ms", round((t1 - t0) * 1e3, 2))
p, o, _ = pr.config("c2b", 4096)
t0 = time.perf_counter(); h = P.homotopy_solve(p, 2, P.IterationOptions(**o)); t1 = time.perf_counter()
print("homotopy c2b n=4096 stages=2:", P.to_string(h.status), h.iterations, "wall_ms", round((t1 - t0) * 1e3, 2))
PY
timeout 600 python /tmp/h.py
