timeout 300 python tools/config_times.py --configs c1 --steps 30 2>&1 | tail -12 | cut -c1-300
