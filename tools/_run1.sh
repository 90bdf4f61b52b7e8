DPT_DENSE_SMALL=5 timeout 300 python tools/config_times.py --configs c1 --steps 50 2>&1 | tail -5 | cut -c1-300
