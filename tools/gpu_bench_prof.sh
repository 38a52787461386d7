mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
cat gpurun_out/bench_full.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:_ZN4dart -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fwd_sweep -s 3 -c 1 -o gpurun_out/prof_fwd -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_fwd.log 2>&1; echo "ncu fwd rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bwd_sweep -s 3 -c 1 -o gpurun_out/prof_bwd -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_bwd.log 2>&1; echo "ncu bwd rc=$?"
