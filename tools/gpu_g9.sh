timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g9_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/g9_pytest.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --head 2>gpurun_out/g9_err.log | tail -1 > gpurun_out/g9_bench_head.json; echo "bench head rc=$?"
timeout 300 python bench.py --no-cpu-baseline --no-e2e --mask causal 2>>gpurun_out/g9_err.log | tail -1 > gpurun_out/g9_bench_causal.json; echo "bench causal rc=$?"
tail -3 gpurun_out/g9_err.log
