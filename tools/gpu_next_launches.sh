export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:_ZN4dart -c 60 --csv --log-file gpurun_out/launches_fused.csv python bench.py --fused --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo fused rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:_ZN4dart -c 60 --csv --log-file gpurun_out/launches_kl.csv python bench.py --kl exact --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo kl rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:_ZN4dart -c 60 --csv --log-file gpurun_out/launches_lmhead.csv python bench.py --lmhead --steps 3 --warmup 3 --no-cpu --no-e2e --no-unfused > /dev/null 2>&1; echo lmhead rc=$?
timeout 600 python bench.py --kl exact --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_kl.json 2>/dev/null; echo klbench rc=$?
