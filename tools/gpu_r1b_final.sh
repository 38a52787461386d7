export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_final.json 2>gpurun_out/bench_final.err; echo "bench rc=$?"; cut -c1-600 gpurun_out/bench_final.json
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_final.json 2>gpurun_out/bench_ref_final.err; echo "ref rc=$?"; cut -c1-300 gpurun_out/bench_ref_final.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:_ZN4dart --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch_final.log 2>&1; echo "ncu rc=$?"
