timeout 900 python -m pytest tests -m gpu -q > gpurun_out/g18_pytest.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/g18_pytest.log
