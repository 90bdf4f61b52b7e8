timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_shim.py -q --timeout 300 -x 2>&1 | tail -2
