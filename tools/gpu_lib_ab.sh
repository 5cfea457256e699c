#!/bin/bash
# A/B of a library variant ($VAR) against libmtgr.so on a config ($CFG, default small): bench x2
mkdir -p gpurun_out
CFG=${CFG:-small}
for r in 1 2; do
  for L in libmtgr.so $VAR; do
    MTGR_LIBRARY=$L timeout 600 python bench.py --config $CFG --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e --no-large-attn > gpurun_out/lab_${CFG}_${L}_$r.json 2> /dev/null
  done
done
