#!/bin/bash
# K3 variant sweep (tuning helper): kernel time of each DPT_U16_VARIANT on c4 / c4b.
for cfg in c4 c4b; do
for v in ${VARIANTS:-0 1 2 3 4 5 6 7 8 9 10}; do
  echo "$cfg variant $v: $(DPT_U16_VARIANT=$v timeout 120 python tools/config_times.py --configs $cfg 2>&1 | head -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["kernel_ms"]*1e3,1), "us", round(d["hbm_frac"],3), d["status"], d["iterations"])')"
done
done
