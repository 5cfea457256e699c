#!/bin/bash
# A/B of the working-tree library against libmtgr_head.so (HEAD): attention parity, then bench x2
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_probe.py -x -q -k "attention or probe or layer_fwd_bwd" > gpurun_out/lab2_parity.log 2>&1; echo "parity rc=$? $(tail -1 gpurun_out/lab2_parity.log)"
for r in 1 2; do
  for L in libmtgr.so libmtgr_head.so; do
    MTGR_LIBRARY=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/lab2_${L}_$r.json 2> /dev/null
  done
done
