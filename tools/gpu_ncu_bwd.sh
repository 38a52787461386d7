mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bwd_sweep -s 3 -c 1 -o gpurun_out/prof_bwd2 -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_bwd2.log 2>&1; echo "ncu bwd rc=$?"
