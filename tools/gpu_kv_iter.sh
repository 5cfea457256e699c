# one iteration on the coupled kernel: parity (kv path), optional trace build, bench
mkdir -p gpurun_out
P=${P:-gx}
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_probe.py -x -q -k "kv" 2>&1 | tail -5 > gpurun_out/${P}_parity.log; echo "parity rc=$?"
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err; echo "bench rc=$?"
if [ -n "$TRACE" ]; then
  make -C paper_2505_18654_b200/csrc -j16 TRACE=1 -B > /dev/null 2>&1
  MTGR_KV_TRACE=1 timeout 300 python tools/kv_trace.py run 2> gpurun_out/${P}_trace.log; echo "trace rc=$?"
fi
