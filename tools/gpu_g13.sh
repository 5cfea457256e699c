mkdir -p gpurun_out
MTGR_KV_DEBUG=16 MTGR_KV_TRACE=1 timeout 300 python tools/kv_trace.py run 2> gpurun_out/g13_trace16.log; echo "trace rc=$?"
MTGR_KV_DEBUG=31 MTGR_KV_TRACE=1 timeout 300 python tools/kv_trace.py run 2> gpurun_out/g13_trace31.log; echo "trace rc=$?"
