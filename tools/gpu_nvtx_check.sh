MTGR_NVTX=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "layer_fwd_bwd and parity and kv" 2>&1 | tail -1
MTGR_NVTX=1 timeout 600 ncu --nvtx --nvtx-include "layer0.bwd/" --metrics gpu__time_duration.sum -c 20 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-large-attn 2>&1 | grep -c "attn_kv\|gemm_tc\|gln_" 
