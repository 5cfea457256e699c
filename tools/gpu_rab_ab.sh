#!/bin/bash
# A/B of the rab bucket variants (libmtgr_bk1 / libmtgr.so = 2 / libmtgr_bk3): rab parity + bench
mkdir -p gpurun_out
for L in libmtgr.so libmtgr_bk1.so libmtgr_bk3.so; do
  MTGR_LIBRARY=$L timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "rab" > gpurun_out/rab_ab_$L.log 2>&1
  echo "$L $(tail -1 gpurun_out/rab_ab_$L.log)"
  MTGR_LIBRARY=$L timeout 400 python bench.py --rab 16 --no-cpu-baseline --no-large-attn --no-e2e > gpurun_out/rab_ab_$L.json 2> gpurun_out/rab_ab_$L.err
done
