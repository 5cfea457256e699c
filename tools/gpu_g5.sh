mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_model.py -x -q 2>&1 | tail -60 > gpurun_out/g5_model.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "attention_fwd_bwd and kv" 2>&1 | tail -30 > gpurun_out/g5_attn.log; echo "attn rc=$?"
timeout 600 python -m pytest tests/test_gpu_probe.py -x -q -k "kv" 2>&1 | tail -30 > gpurun_out/g5_probe.log; echo "probe rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "kv" 2>&1 | tail -30 > gpurun_out/g5_parity.log; echo "parity rc=$?"
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/g5_bench.json 2> gpurun_out/g5_bench.err; echo "bench rc=$?"
