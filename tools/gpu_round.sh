set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/g1_pytest.log
timeout 300 python bench.py > gpurun_out/g1_bench_small.json 2> gpurun_out/g1_bench_small.err; echo "bench rc=$?"
timeout 600 python bench.py --config large --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g1_bench_large.json 2> gpurun_out/g1_bench_large.err; echo "bench large rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/g1_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/g1_ncu.log 2>&1; echo "ncu rc=$?"
