mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stream_gpu.py -q --timeout 600 > gpurun_out/pytest_stream.log 2>&1; echo "stream pytest rc=$?"; tail -5 gpurun_out/pytest_stream.log
timeout 900 python bench.py --config long --stream-rows 32768 --pool 3 --steps 3 --warmup 3 > gpurun_out/bench_long.json 2> gpurun_out/bench_long.err; echo "long rc=$?"; cat gpurun_out/bench_long.json; tail -3 gpurun_out/bench_long.err
