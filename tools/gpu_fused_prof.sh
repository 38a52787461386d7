mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
DART_FUSED_VARIANT=${VARIANT:-1} timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_cluster -s 2 -c 1 -o gpurun_out/prof_fused_cl -f python bench.py --fused --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_fused_cl.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_fused_cl.log
