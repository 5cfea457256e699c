# compute-sanitizer (memcheck, racecheck, synccheck) over every tensor-core path on small batches
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for path in kv stored fused_dk recompute; do
    if [ $path = recompute ]; then env="MTGR_ATTN_RECOMPUTE=1"; else env="MTGR_ATTN_BWD=$path"; fi
    env $env timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_run.py toy parity \
      > gpurun_out/sanitize/${tool}_${path}.log 2>&1
    echo "$tool $path rc=$?"
  done
done
