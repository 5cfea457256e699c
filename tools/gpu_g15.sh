mkdir -p gpurun_out
for dbg in 0 1 2 4 3 7; do
MTGR_KV_DEBUG=$dbg MTGR_KV_TRACE=1 timeout 300 python tools/kv_trace.py run 2> gpurun_out/g15_trace_d$dbg.log; echo "trace $dbg rc=$?"
done
