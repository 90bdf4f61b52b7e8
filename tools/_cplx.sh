timeout 300 python tools/config_times.py --configs c4,c4b --complex > gpurun_out/cplx_w10.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_k3_variants.py -x -q -k complex > gpurun_out/cplx_w10_test.log 2>&1
