#!/bin/bash
# ncu of the rab kernels (drab, FWD with RAB) at `small` with --rab 16
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_drab_kernel" -c 1 \
  -o gpurun_out/r02_drab python bench.py --rab 16 --no-cpu-baseline --no-large-attn --no-e2e --steps 1 --warmup 0 \
  > gpurun_out/r02_drab_ncu.log 2>&1
tail -3 gpurun_out/r02_drab_ncu.log
