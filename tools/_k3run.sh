timeout 600 python -m pytest tests/test_gpu_staged_io.py tests/test_gpu_k3_variants.py tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py -x -q > gpurun_out/k3r_test.log 2>&1
VARIANTS="1 11 16" bash tools/u16_sweep.sh > gpurun_out/k3r_sweep.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:single_u16 -s 1 -c 1 -o gpurun_out/k3_rot -f python tools/profile_run.py --config c4 --steps 3 > gpurun_out/k3_ncu_rot.log 2>&1
