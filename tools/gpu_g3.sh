timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "attention or layer_fwd_bwd or edge" > gpurun_out/g3_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/g3_parity.log
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/g3_bench_small_$i.json; echo "bench rc=$?"
MTGR_ATTN_RECOMPUTE=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/g3_bench_small_rc_$i.json; echo "bench rc=$?"
done
