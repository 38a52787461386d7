mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multirank_gpu.py -q --timeout 600 > gpurun_out/pytest_mr.log 2>&1; echo "mr pytest rc=$?"; tail -15 gpurun_out/pytest_mr.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --backend gloo --no-e2e > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err; echo "bench2 rc=$?"; cat gpurun_out/bench_2rank.json; tail -5 gpurun_out/bench_2rank.err
