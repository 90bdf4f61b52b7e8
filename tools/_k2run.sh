timeout 300 python tools/config_times.py --configs c3 > gpurun_out/k2_cfg.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_csr_paths.py tests/test_gpu_csr_schedules.py -x -q > gpurun_out/k2_test.log 2>&1
