export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_phases.json 2>gpurun_out/bench_phases.err; echo "rc=$?"; python -c "
import json; j=json.load(open('gpurun_out/bench_phases.json')); print(j['value'], j['kernels']['phases_median_ms'])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --backend gloo --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_2rank_gloo.json 2>gpurun_out/bench_2rank_gloo.err; echo "2rank rc=$?"; python -c "
import json; j=json.load(open('gpurun_out/bench_2rank_gloo.json')); print(j['value'], j['n_gpus'], j['kernels']['phases_median_ms'], j['e2e'])"; tail -3 gpurun_out/bench_2rank_gloo.err
