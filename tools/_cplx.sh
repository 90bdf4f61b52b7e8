timeout 300 python tools/config_times.py --configs c4,c4b --complex > gpurun_out/cplx_u16.jsonl 2>&1
DPT_CPLX_U16=0 timeout 300 python tools/config_times.py --configs c4,c4b --complex > gpurun_out/cplx_gen.jsonl 2>&1
timeout 300 python tools/config_times.py --configs c4,c4b > gpurun_out/real_u16.jsonl 2>&1
