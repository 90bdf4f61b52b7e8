set -x
timeout 600 python bench.py > gpurun_out/bench_final.log 2>&1; tail -1 gpurun_out/bench_final.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py > gpurun_out/ncu_bench.log 2>&1; tail -2 gpurun_out/ncu_bench.log
DPT_GRAPH_LOOP=0 timeout 600 ncu --kernel-name regex:csr_step --launch-skip 2 --launch-count 1 --clock-control none --set full --import-source on -o gpurun_out/prof_csr_c3 -f python tools/profile_run.py --config c3 --steps 4 > gpurun_out/ncu_csr.log 2>&1; tail -1 gpurun_out/ncu_csr.log
DPT_GRAPH_LOOP=0 timeout 600 ncu --kernel-name regex:dense_step --launch-skip 2 --launch-count 1 --clock-control none --set full --import-source on -o gpurun_out/prof_dense_c2 -f python tools/profile_run.py --config c2 --steps 4 > gpurun_out/ncu_dense.log 2>&1; tail -1 gpurun_out/ncu_dense.log
DPT_GRAPH_LOOP=0 timeout 600 ncu --kernel-name regex:single_u16 --launch-skip 2 --launch-count 1 --clock-control none --set full --import-source on -o gpurun_out/prof_single_c4 -f python tools/profile_run.py --config c4 --steps 4 > gpurun_out/ncu_single.log 2>&1; tail -1 gpurun_out/ncu_single.log
cat > /tmp/sc.py <<'PY'
import sys; sys.path.insert(0, ".")
import paper_2002_12872_b200 as P
from paper_2002_12872_b200 import problems as pr
from paper_2002_12872_b200.dpt import ScanGrid, ScanMode, IterationOptions, PartitionedProblem
P.scan_domain(pr.two_by_two(1.0), ScanGrid(-1.2, 1.2, -1.0, 1.0, 512, 512), ScanMode("Full", 0), IterationOptions(max_iter=300))
P.scan_domain(PartitionedProblem(*pr.random_uniform(6, 3), 0.0), ScanGrid(-0.4, 0.4, -0.3, 0.3, 512, 512), ScanMode("Full", 0), IterationOptions(max_iter=300))
PY
timeout 600 ncu --kernel-name regex:scan_ --clock-control none --set full --import-source on -o gpurun_out/prof_scan -f python /tmp/sc.py > gpurun_out/ncu_scan.log 2>&1; tail -1 gpurun_out/ncu_scan.log
