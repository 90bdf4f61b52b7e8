timeout 900 python -m pytest tests/test_gpu_edge.py -q --timeout 300 -x 2>&1 | grep -v "^  File" | tail -30
