export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 --maxfail 40 > gpurun_out/pytest_gpu_r1b.log 2>&1; echo "pytest rc=$?"
tail -8 gpurun_out/pytest_gpu_r1b.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_r1b.json 2>gpurun_out/bench_r1b.err; echo "bench rc=$?"; cat gpurun_out/bench_r1b.json
