for c in 0 1 2 3 4 5; do echo "cfg $c"; DPT_CSR_CFG=$c timeout 300 python tools/config_times.py --configs c3 2>&1 | cut -c1-200; done > gpurun_out/k2_cfg.txt
echo "unpaired cfg 0" >> gpurun_out/k2_cfg.txt; DPT_SELL_PAIR=0 timeout 300 python tools/config_times.py --configs c3 2>&1 | cut -c1-200 >> gpurun_out/k2_cfg.txt
timeout 300 python tools/config_times.py --configs c3 --complex 2>&1 | cut -c1-200 >> gpurun_out/k2_cfg.txt
timeout 600 python -m pytest tests/test_gpu_csr_paths.py tests/test_gpu_csr_schedules.py -x -q > gpurun_out/k2_test.log 2>&1
