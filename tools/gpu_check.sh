mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 --maxfail 30 -x -k "tiny or small_multi or selection or odd or zero_fill or status or bad_meta or neg_inf" > gpurun_out/pytest_gpu1.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu1.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?"
cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
