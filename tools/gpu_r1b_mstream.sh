export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_multirank_gpu.py -m gpu -q -x > gpurun_out/pytest_mstream.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_mstream.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --backend gloo --config adaptive --stream-rows 16384 --pool 2 --steps 3 --warmup 3 > gpurun_out/bench_mstream_gloo.json 2>gpurun_out/bench_mstream_gloo.err; echo "mstream rc=$?"; cut -c1-400 gpurun_out/bench_mstream_gloo.json; tail -3 gpurun_out/bench_mstream_gloo.err
timeout 900 python bench.py --config long --stream-rows 32768 --steps 2 --warmup 3 > gpurun_out/bench_stream_long_r1b.json 2>gpurun_out/bench_stream_long_r1b.err; echo "long rc=$?"; python -c "
import json; j=json.load(open('gpurun_out/bench_stream_long_r1b.json')); print(j['value'], j['roofline']['frac'], j['clocks'])"
