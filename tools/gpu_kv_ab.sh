#!/bin/bash
# coupled-kernel change: kv parity / probes / guards, then A/B bench against libmtgr_head.so
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "kv and (attention or layer_fwd_bwd or ablation or rab)" > gpurun_out/kab_parity.log 2>&1; echo "parity rc=$? $(tail -1 gpurun_out/kab_parity.log)"
timeout 300 python -m pytest tests/test_gpu_probe.py tests/test_gpu_guards.py -x -q -k "kv" > gpurun_out/kab_probe.log 2>&1; echo "probe rc=$? $(tail -1 gpurun_out/kab_probe.log)"
for r in 1 2; do
  for L in libmtgr.so libmtgr_head.so; do
    MTGR_LIBRARY=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/kab_${L}_$r.json 2> /dev/null
    echo "$L $r $?"
  done
done
