timeout 900 python -m pytest tests/test_gpu_dense_paths.py -q --timeout 600 -x 2>&1 | grep -v "^  File" | tail -15
