export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
bash tools/gpu_configs.sh
timeout 600 python bench.py --fused --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_fused_s2.json 2>/dev/null; echo "fused rc=$?"; python -c "
import json; j=json.load(open('gpurun_out/bench_fused_s2.json')); print('fused', j['value'], j['roofline']['frac'], j['clocks']['sm_mhz'])"
timeout 600 python bench.py --kl exact --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_kl_s2.json 2>/dev/null; echo "kl rc=$?"; python -c "
import json; j=json.load(open('gpurun_out/bench_kl_s2.json')); print('kl', j['value'], j['kernels']['step_frac'], j['clocks']['sm_mhz'])"
timeout 900 python bench.py --lmhead --steps 10 --warmup 3 > gpurun_out/bench_lmhead_s2.json 2>/dev/null; echo "lmhead rc=$?"; python -c "
import json; j=json.load(open('gpurun_out/bench_lmhead_s2.json')); print('lmhead', j['value'], j['roofline']['achieved'], j['roofline']['frac'], j['clocks']['sm_mhz'], (j.get('unfused_cublas_pipeline') or {}).get('ms_per_step'), j['ms_per_step'])"
