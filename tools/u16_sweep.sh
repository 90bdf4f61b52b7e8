#!/bin/bash
# K3 variant sweep (tuning helper): kernel time of each DPT_U16_VARIANT on c4.
for v in 0 1 2 3 4 5; do
  echo "variant $v: $(DPT_U16_VARIANT=$v timeout 120 python tools/config_times.py --configs c4 2>&1 | head -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["kernel_ms"], d["status"], d["iterations"])')"
done
