timeout 600 python -m pytest tests/test_gpu_embed.py -x -q > gpurun_out/g11_embed.log 2>&1; echo "embed rc=$?"; tail -30 gpurun_out/g11_embed.log
timeout 300 python bench_embed.py > gpurun_out/g11_bench_embed.json 2> gpurun_out/g11_bench_embed.err; echo "bench embed rc=$?"; tail -2 gpurun_out/g11_bench_embed.json; tail -5 gpurun_out/g11_bench_embed.err
