mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 --maxfail 40 > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu2.log
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fwd_sweep -s 2 -c 1 -o gpurun_out/prof_fwd -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_fwd.log 2>&1; echo "ncu fwd rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bwd_sweep -s 2 -c 1 -o gpurun_out/prof_bwd -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_bwd.log 2>&1; echo "ncu bwd rc=$?"
ls -la gpurun_out/
