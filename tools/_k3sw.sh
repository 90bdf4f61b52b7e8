VARIANTS="11 15 16 17 18" bash tools/u16_sweep.sh > gpurun_out/k3v_sweep3.txt 2>&1
echo "carveout 100" >> gpurun_out/k3v_sweep3.txt
DPT_U16_CARVEOUT=100 VARIANTS="6 11 15 16 17 18" bash tools/u16_sweep.sh >> gpurun_out/k3v_sweep3.txt 2>&1
