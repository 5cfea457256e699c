mkdir -p gpurun_out
for dbg in 0 32 16; do
MTGR_KV_DEBUG=$dbg timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-large-attn --steps 5 > gpurun_out/g30_d$dbg.json 2>> gpurun_out/g30.err; echo "dbg $dbg rc=$?"
done
