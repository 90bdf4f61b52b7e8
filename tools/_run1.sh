timeout 1200 python -m pytest tests/test_gpu_fuzz.py -q --timeout 300 2>&1 | tail -25
