DPT_TIMING=1 timeout 120 python tools/c4b_solve.py > gpurun_out/c4b_timing.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/lv_pytest.log 2>&1
