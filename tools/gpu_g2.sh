timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "attention or layer_fwd_bwd or edge" > gpurun_out/g2_parity.log 2>&1; echo "parity rc=$?"; tail -5 gpurun_out/g2_parity.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/g2_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/g2_pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/g2_bench_small.json 2> gpurun_out/g2_bench_small.err; echo "bench rc=$?"
timeout 600 python bench.py --config large --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g2_bench_large.json 2> gpurun_out/g2_bench_large.err; echo "bench large rc=$?"
