# A/B of library builds on one box: libmtgr.so (current) vs libmtgr_head.so (last commit)
mkdir -p gpurun_out
P=${P:-ab}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_probe.py -x -q -k "attention_fwd_bwd or layer_fwd_bwd or probe" 2>&1 | tail -3 > gpurun_out/${P}_parity.log; echo "parity rc=$?"
for i in 1 2; do for L in libmtgr.so libmtgr_head.so; do
  MTGR_LIBRARY=$L timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-large-attn > gpurun_out/${P}_${L}_$i.json 2>> gpurun_out/${P}_bench.err
done; done
for L in libmtgr.so libmtgr_head.so; do
  MTGR_LIBRARY=$L timeout 300 python bench.py --config large --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${P}_${L}_large.json 2>> gpurun_out/${P}_bench.err
done
