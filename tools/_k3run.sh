set -x
timeout 300 python -m pytest tests/test_gpu_k3_variants.py tests/test_gpu_parity.py -x -q -k "k3 or c4" > gpurun_out/k3v_test.log 2>&1
timeout 300 python tools/config_times.py --configs c4,c4b,c3 > gpurun_out/k3_cfg.jsonl 2>&1
for r in 2 1; do DPT_CSR_ROWS=$r timeout 300 python tools/config_times.py --configs c3 >> gpurun_out/k3_cfg.jsonl 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:single_u16 -s 1 -c 1 -o gpurun_out/k3_v11 -f python tools/profile_run.py --config c4 --steps 3 > gpurun_out/k3_ncu_v11.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k3_launches_c4.csv python tools/profile_run.py --config c4 --steps 6 > /dev/null 2>&1
