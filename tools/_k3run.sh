set -x
timeout 300 python -m pytest tests/test_gpu_k3_variants.py -x -q > gpurun_out/k3v_test.log 2>&1
for v in 1 10; do
DPT_U16_VARIANT=$v timeout 300 python tools/profile_run.py --config c4 --steps 3 > /dev/null 2>&1 && \
DPT_U16_VARIANT=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:single_u16 -s 1 -c 1 -o gpurun_out/k3_v$v -f python tools/profile_run.py --config c4 --steps 3 > gpurun_out/k3_ncu_v$v.log 2>&1
done
