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
timeout 600 python -m pytest tests/test_gpu_staged_io.py tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_shim.py -x -q > gpurun_out/sel_pytest.log 2>&1
DPT_TIMING=1 timeout 300 python /tmp/ph.py > gpurun_out/phase3.txt 2>&1
timeout 600 python tools/host_wall.py --configs c4,c4b > gpurun_out/host_wall_sel.jsonl 2>&1
