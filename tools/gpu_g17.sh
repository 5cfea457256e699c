timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g17_pytest.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/g17_pytest.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --post-mlp 2 2>/dev/null | tail -1 > gpurun_out/g17_bench_post2.json; echo "bench rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g17_smoke.log 2>&1; echo "smoke rc=$?"
