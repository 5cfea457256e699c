# round-end evidence: tests, smoke, bench lines, ncu launch list and full captures
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?"
timeout 400 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?"
timeout 400 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/f_bench_ref.json 2>> gpurun_out/f_bench.err; echo "ref rc=$?"
timeout 400 python bench.py --tokens --head --no-e2e --no-cpu-baseline > gpurun_out/f_bench_full_model.json 2>> gpurun_out/f_bench.err; echo "full-model rc=$?"
timeout 600 python bench.py --config large --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_bench_large.json 2>> gpurun_out/f_bench.err; echo "large rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/f_ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_mm_kernel|attn_tc_kernel|attn_sc_kernel" --launch-skip 2 -c 5 -o gpurun_out/f_attn python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_ncu_attn.log 2>&1; echo "ncu attn rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc_kernel|gln_" --launch-skip 10 -c 10 -o gpurun_out/f_other python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_ncu_other.log 2>&1; echo "ncu other rc=$?"
tail -3 gpurun_out/f_bench.err
