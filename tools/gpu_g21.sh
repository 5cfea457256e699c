mkdir -p gpurun_out
for sl in 32 256 1024 4096; do
MTGR_KV_SLEEP=$sl timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-large-attn > gpurun_out/g21_sleep$sl.json 2>> gpurun_out/g21.err; echo "sleep $sl rc=$?"
done
