#!/bin/bash
# ncu --set full of the QKVU GEMM (gemm_tc_kernel<1, 2>) at `small`
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel --launch-skip 0 -c 1 \
  -o gpurun_out/qkvu python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-large-attn > gpurun_out/qkvu_ncu.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/qkvu_ncu.log
