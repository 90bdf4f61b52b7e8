VARIANTS="11 19 20" bash tools/u16_sweep.sh > gpurun_out/k3v_sweep4.txt 2>&1
for c in 44 50; do echo "carveout $c" >> gpurun_out/k3v_sweep4.txt; DPT_U16_CARVEOUT=$c VARIANTS="11 19" bash tools/u16_sweep.sh >> gpurun_out/k3v_sweep4.txt 2>&1; done
timeout 300 python -m pytest tests/test_gpu_k3_variants.py -x -q > gpurun_out/k3v_test2.log 2>&1
