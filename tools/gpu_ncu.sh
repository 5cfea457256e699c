# ncu evidence for profiles/: launch list of the default bench (cold, serialised) and full
# captures of the top kernels at `small` and of the attention kernels at MTGR-large
mkdir -p gpurun_out
P=${P:-nc}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${P}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-large-attn > gpurun_out/${P}_ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"attn_kv_kernel|attn_tc_kernel|attn_mm_kernel" --launch-skip 3 -c 3 -o gpurun_out/${P}_attn_small python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-large-attn > gpurun_out/${P}_ncu_attn.log 2>&1; echo "ncu attn rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc_kernel|gln_" --launch-skip 10 -c 8 -o gpurun_out/${P}_other_small python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-large-attn > gpurun_out/${P}_ncu_other.log 2>&1; echo "ncu other rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"attn_kv_kernel|attn_tc_kernel|attn_mm_kernel" --launch-skip 3 -c 3 -o gpurun_out/${P}_attn_large python bench.py --config large --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${P}_ncu_large.log 2>&1; echo "ncu large rc=$?"
