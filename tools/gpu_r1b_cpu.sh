export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
nproc; free -g | head -2; lscpu | grep "Model name"
timeout 900 python bench.py > gpurun_out/bench_r1c.json 2>gpurun_out/bench_r1c.err; echo "bench rc=$?"; python -c "
import json; j=json.load(open('gpurun_out/bench_r1c.json')); print(j['value'], j['kernels']['step_frac'], j['clocks'], j['cpu_baseline'], j.get('copy_sustained',{}).get('GBps'), j['e2e'])"
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_r1c.json 2>gpurun_out/bench_ref_r1c.err; echo "ref rc=$?"; cat gpurun_out/bench_ref_r1c.json | cut -c1-300
