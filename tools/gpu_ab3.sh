# A/B: libmtgr.so (double-buffered coupled kernel) vs libmtgr_ns3.so (triple) vs stored path
mkdir -p gpurun_out
P=${P:-ab3}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_probe.py -x -q -k "kv" 2>&1 | tail -3 > gpurun_out/${P}_parity.log; echo "parity rc=$?"
for i in 1 2; do
  for L in libmtgr.so libmtgr_head.so; do
    MTGR_LIBRARY=$L timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-large-attn > gpurun_out/${P}_${L}_$i.json 2>> gpurun_out/${P}_bench.err
  done
  MTGR_ATTN_BWD=stored timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-large-attn > gpurun_out/${P}_stored_$i.json 2>> gpurun_out/${P}_bench.err
done
