timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -4
for c in c1 c4 c4b c3 c2b; do timeout 120 python tools/kineto_trace.py --config $c --json gpurun_out/kineto_$c.json 2>&1 | grep -v Warn | grep -v warn_once; done
timeout 300 python tools/solve_wall.py --configs c1,c3,c4,c4b,c2b --reps 4 2>&1 | tee gpurun_out/solve_wall.txt
