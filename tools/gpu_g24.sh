mkdir -p gpurun_out
for dbg in 0 8 9 16 24 25 31; do
MTGR_KV_DEBUG=$dbg timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-large-attn --steps 5 > gpurun_out/g24_d$dbg.json 2>> gpurun_out/g24.err; echo "dbg $dbg rc=$?"
done
