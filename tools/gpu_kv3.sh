#!/bin/bash
# A/B of coupled-kernel build variants: kv parity on the first variant, then bench x2 each
mkdir -p gpurun_out
V1=${V1:-libmtgr_c1.so}; V2=${V2:-libmtgr_c3.so}
MTGR_LIBRARY=$V2 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "kv and (attention or layer_fwd_bwd)" 2>&1 | tail -1
for r in 1 2; do for L in libmtgr.so $V1 $V2; do
  MTGR_LIBRARY=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/k3_${L}_$r.json 2> /dev/null; done; done
