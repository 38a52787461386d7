# ncu evidence of the bench's kernels (outputs gpurun_out/launches.csv, prof_{fwd,bwd,fused}.ncu-rep);
# then, here: python tools/summarize_profiles.py <tag>
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:_ZN4dart -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fwd_sweep -s 3 -c 1 -o gpurun_out/prof_fwd -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_fwd.log 2>&1; echo "ncu fwd rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bwd_sweep -s 3 -c 1 -o gpurun_out/prof_bwd -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_bwd.log 2>&1; echo "ncu bwd rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fused_sweep -s 1 -c 1 -o gpurun_out/prof_fused -f python bench.py --fused --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_fused.log 2>&1; echo "ncu fused rc=$?"
