timeout 600 python -m pytest tests/test_gpu_head.py -x -q > gpurun_out/g8_head.log 2>&1; echo "head rc=$?"; tail -30 gpurun_out/g8_head.log
