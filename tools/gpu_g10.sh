timeout 600 python -m pytest tests/test_gpu_token.py -x -q > gpurun_out/g10_token.log 2>&1; echo "token rc=$?"; tail -30 gpurun_out/g10_token.log
