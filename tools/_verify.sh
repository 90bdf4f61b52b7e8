set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/v_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/v_smoke.log
timeout 600 python bench.py > gpurun_out/v_bench.jsonl 2> gpurun_out/v_bench.err; echo "bench rc=$?" >> gpurun_out/v_bench.err
timeout 1200 python bench.py --baselines > gpurun_out/v_baselines.jsonl 2> gpurun_out/v_baselines.err
tail -3 gpurun_out/v_pytest.log
