set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/v_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/v_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/v_smoke.log
timeout 600 python bench.py > gpurun_out/v_bench.jsonl 2> gpurun_out/v_bench.err; echo "bench rc=$?" >> gpurun_out/v_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/v_bench_ref.jsonl 2> gpurun_out/v_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-calls 1 > gpurun_out/v_ncu_bench.log 2>&1
tail -3 gpurun_out/v_pytest.log
