# A/B of the coupled dK/dV kernel's coupling costs (MTGR_KV_DEBUG bits: timing only) + ncu capture
mkdir -p gpurun_out
P=${P:-g6}
for dbg in 0 1 2 4 7 15; do
  MTGR_KV_DEBUG=$dbg timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-large-attn > gpurun_out/${P}_bench_dbg$dbg.json 2>> gpurun_out/${P}_bench.err
  echo "dbg=$dbg rc=$?"
done
MTGR_ATTN_BWD=stored timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-large-attn > gpurun_out/${P}_bench_stored.json 2>> gpurun_out/${P}_bench.err
timeout 600 python -m pytest tests/test_gpu_model.py -q -x 2>&1 | tail -3 > gpurun_out/${P}_model.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_kv_kernel" --launch-skip 3 -c 1 -o gpurun_out/${P}_kv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-large-attn > gpurun_out/${P}_ncu.log 2>&1; echo "ncu rc=$?"
