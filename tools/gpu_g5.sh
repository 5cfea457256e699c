# 4-GPU scaling evidence: small (weak scaling, the bench workload), middle and large_skew (LPT-balanced DP)
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 ${@:3} 2> gpurun_out/g5_err_$2.log | tail -1; }
python bench.py --config large --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/g5_large_n1.json
run 4 29510 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/g5_small_n4.json
run 2 29511 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g5_small_n2.json
run 4 29512 --config middle --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g5_middle_n4.json
python bench.py --config middle --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/g5_middle_n1.json
run 4 29513 --config large_skew --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g5_large_skew_n4.json
ls -la gpurun_out/
