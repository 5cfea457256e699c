#!/bin/bash
mkdir -p gpurun_out
for r in 1 2; do
  for L in libmtgr.so libmtgr_r2.so; do
    MTGR_LIBRARY=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-large-attn > gpurun_out/ring_${L}_$r.json 2> /dev/null
  done
done
