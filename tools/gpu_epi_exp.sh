#!/bin/bash
mkdir -p gpurun_out
for r in 1 2; do
  for L in libmtgr.so libmtgr_e1.so libmtgr_e2.so libmtgr_e3.so; do
    MTGR_LIBRARY=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-large-attn > gpurun_out/epi_${L}_$r.json 2> /dev/null
  done
done
