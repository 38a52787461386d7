mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fused_sweep -s 2 -c 1 -o gpurun_out/prof_fused -f python bench.py --fused --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_fused.log 2>&1; echo "ncu fused rc=$?"
