for g in 16 32; do
DPT_SELL_GROUP=$g timeout 300 python tools/config_times.py --configs c3 --steps 20 2>&1 | head -1
DPT_SELL_GROUP=$g timeout 300 ncu --kernel-name regex:csr_step --launch-skip 2 --launch-count 1 --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum python tools/profile_run.py --config c3 --steps 4 2>&1 | tail -9
done
