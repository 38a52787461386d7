mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python -m pytest tests/test_fused_gpu.py -x -q 2>&1 | tail -15
for v in 1 0; do
DART_FUSED_VARIANT=$v timeout 600 python bench.py --fused --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_fused_v$v.json 2> gpurun_out/bench_fused_v$v.err; echo "variant $v rc=$?"
python -c "
import json; j=json.load(open('gpurun_out/bench_fused_v$v.json'))
print('variant $v', round(j['value']/1e6,3), 'M tok/s', j['ms_per_step'], 'ms', j['roofline']['frac'], j['clocks'])"
done
