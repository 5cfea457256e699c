#!/bin/bash
# half-tile kv kernel: parity subsets, then A/B bench against libmtgr_head.so (previous build)
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "kv and (attention or layer_fwd_bwd or ablation)" > gpurun_out/ht_parity.log 2>&1; echo "parity rc=$? $(tail -1 gpurun_out/ht_parity.log)"
timeout 400 python -m pytest tests/test_gpu_probe.py tests/test_gpu_guards.py -x -q -k "kv" > gpurun_out/ht_probe.log 2>&1; echo "probe rc=$? $(tail -1 gpurun_out/ht_probe.log)"
for r in 1 2; do
  for L in libmtgr.so libmtgr_head.so; do
    MTGR_LIBRARY=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ht_ab_${L}_$r.json 2> /dev/null
    echo "$L $r $?"
  done
done
