export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_lmhead_update_gpu.py -m gpu -q -x 2>&1 | tail -1
for g in 2 1 4 2 1 4; do timeout 600 python bench.py --lmhead --update --steps 5 --warmup 3 --no-unfused --dw-group $g > gpurun_out/bench_lmup_g.json 2>/dev/null; python -c "
import json; j=json.load(open('gpurun_out/bench_lmup_g.json')); print('dw_group=$g', j['ms_per_step'], round(j['roofline']['achieved']), j['clocks']['sm_mhz'])"; done
