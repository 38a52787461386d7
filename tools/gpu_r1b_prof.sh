export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_copyref.json 2>gpurun_out/bench_copyref.err; echo "bench rc=$?"; cat gpurun_out/bench_copyref.json
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fwd_sweep -s 2 -c 1 -o gpurun_out/prof_fwd_b -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_fwd_b.log 2>&1; echo "ncu fwd rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bwd_sweep -s 2 -c 1 -o gpurun_out/prof_bwd_b -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_bwd_b.log 2>&1; echo "ncu bwd rc=$?"
ls -la gpurun_out/
