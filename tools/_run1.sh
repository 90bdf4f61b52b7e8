timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_complex.py tests/test_gpu_shim.py -q --timeout 300 -x -k "csr or c3 or CSR or sparse or complex or shim" 2>&1 | tail -3
timeout 300 python tools/solve_wall.py --configs c3 --reps 4 2>&1
timeout 300 python tools/config_times.py --configs c3 --steps 20 2>&1 | head -1
DPT_GRAPH_LOOP=0 timeout 300 ncu --kernel-name regex:csr_step --launch-skip 2 --launch-count 1 --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum python tools/profile_run.py --config c3 --steps 4 2>&1 | tail -5
