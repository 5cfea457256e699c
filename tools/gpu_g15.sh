timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "attention or layer_fwd_bwd or causal or edge" > gpurun_out/g15_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/g15_parity.log
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>gpurun_out/g15_err.log | tail -1 > gpurun_out/g15_bench_$i.json; echo "bench rc=$?"
done
