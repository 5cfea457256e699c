# round-end evidence: tests, smoke, bench lines, ncu launch list and full captures
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?"
timeout 400 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?"
timeout 400 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/f_bench_ref.json 2>> gpurun_out/f_bench.err; echo "ref rc=$?"
timeout 400 python bench.py --rab 16 --no-cpu-baseline --no-large-attn > gpurun_out/f_bench_rab16.json 2>> gpurun_out/f_bench.err; echo "rab rc=$?"
timeout 400 python bench.py --tokens --head --no-e2e --no-cpu-baseline --no-large-attn > gpurun_out/f_bench_full_model.json 2>> gpurun_out/f_bench.err; echo "full-model rc=$?"
timeout 600 python bench.py --config large --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-large-attn > gpurun_out/f_bench_large.json 2>> gpurun_out/f_bench.err; echo "large rc=$?"
timeout 300 python bench_infer.py > gpurun_out/f_bench_infer.jsonl 2>> gpurun_out/f_bench.err; echo "infer rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-large-attn > gpurun_out/f_ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_kv_kernel|attn_mm_kernel|attn_tc_kernel" --launch-skip 3 -c 3 -o gpurun_out/f_attn python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-large-attn > gpurun_out/f_ncu_attn.log 2>&1; echo "ncu attn rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc_kernel|gln_" --launch-skip 10 -c 10 -o gpurun_out/f_other python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-large-attn > gpurun_out/f_ncu_other.log 2>&1; echo "ncu other rc=$?"
tail -3 gpurun_out/f_bench.err
