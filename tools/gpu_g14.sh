mkdir -p gpurun_out
for ng in 8 16 32; do
MTGR_KV_NG=$ng MTGR_KV_TRACE=1 timeout 300 python tools/kv_trace.py run 2> gpurun_out/g14_trace_ng$ng.log; echo "trace rc=$?"
done
MTGR_KV_DEBUG=16 MTGR_KV_NG=32 MTGR_KV_TRACE=1 timeout 300 python tools/kv_trace.py run 2> gpurun_out/g14_trace_ng32_d16.log
for ng in 8 16 32; do
MTGR_KV_NG=$ng timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-large-attn > gpurun_out/g14_bench_ng$ng.json 2>> gpurun_out/g14_bench.err; echo "bench rc=$?"
done
