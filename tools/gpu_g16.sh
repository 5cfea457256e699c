MTGR_SC_NOSTORE=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/g16_nostore.json
timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/g16_base.json
