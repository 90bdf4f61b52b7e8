#!/bin/bash
# Round-2 ncu captures (run under gpurun, one GPU): full sets of the hot kernels
# and the bench launch list.  Summarise here with tools/ncu_summary.py.
set -x
O=gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:dense_step_kernel -s 2 -c 1 -f -o $O/prof_dense_c2 python tools/profile_run.py --config c2 --steps 4 > $O/prof_dense_c2.log 2>&1
$NCU -k regex:dense_step_kernel -s 2 -c 1 -f -o $O/prof_dense_c1 python tools/profile_run.py --config c1 --steps 4 > $O/prof_dense_c1.log 2>&1
$NCU -k regex:csr_step_kernel -s 2 -c 1 -f -o $O/prof_csr_c3 python tools/profile_run.py --config c3 --steps 4 > $O/prof_csr_c3.log 2>&1
$NCU -k regex:single_u16w -s 2 -c 1 -f -o $O/prof_single_c4 python tools/profile_run.py --config c4 --steps 4 > $O/prof_single_c4.log 2>&1
$NCU -k regex:gemm_nt_kernel -c 1 -f -o $O/prof_gemm_4096 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, paper_2002_12872_b200 as P
r=np.random.default_rng(0); a=r.standard_normal((4096,4096)); P.matmul_dense(a,a)" > $O/prof_gemm.log 2>&1
$NCU -k regex:lu_panel_kernel -c 1 -f -o $O/prof_lu_panel_4096 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, paper_2002_12872_b200 as P
r=np.random.default_rng(0); a=r.standard_normal((4096,4096))+200*np.eye(4096); P.solve_linear_multi(a,a[:, :8])" > $O/prof_lu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02_launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --e2e-calls 1 --no-cpu-baseline > $O/r02_launches_bench.log 2>&1
ls -la $O/*.ncu-rep
