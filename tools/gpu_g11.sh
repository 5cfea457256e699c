mkdir -p gpurun_out
MTGR_KV_TRACE=1 timeout 300 python tools/kv_trace.py run 2> gpurun_out/g11_trace.log; echo "trace rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gln or layer_fwd_bwd" 2>&1 | tail -3 > gpurun_out/g11_gln.log; echo "gln rc=$?"
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-large-attn > gpurun_out/g11_bench.json 2> gpurun_out/g11_bench.err; echo "bench rc=$?"
