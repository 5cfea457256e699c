timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/g13_parity.log 2>&1; echo "parity rc=$?"; tail -15 gpurun_out/g13_parity.log
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>gpurun_out/g13_err.log | tail -1 > gpurun_out/g13_bench_$i.json; echo "bench rc=$?"
MTGR_ATTN_FUSED_DK=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>>gpurun_out/g13_err.log | tail -1 > gpurun_out/g13_bench_fused_$i.json; echo "bench rc=$?"
done
tail -3 gpurun_out/g13_err.log
