export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_graph_gpu.py -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py --graph --no-cpu --no-e2e > gpurun_out/bench_graph.json 2>gpurun_out/bench_graph.err; echo "rc=$?"; python -c "
import json; j=json.load(open('gpurun_out/bench_graph.json')); print(j['value'], j['ms_per_step'], j.get('cuda_graph'), j['clocks'])"; tail -3 gpurun_out/bench_graph.err
