mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests/test_fused_gpu.py -q --timeout 900 > gpurun_out/pytest_fused.log 2>&1; echo "fused pytest rc=$?"; tail -15 gpurun_out/pytest_fused.log
for i in 1 2; do timeout 300 python bench.py --fused --steps 30 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('fused', round(d['value']/1e6,3),'Mtok/s', 'kernel', round(k['bwd_sweep']['frac'],3), round(k['bwd_sweep']['avg_ms'],3), 'step', round(k['step_frac'],3), d['ms_per_step'], d['clocks'])"; done
timeout 1200 ncu --set full --clock-control none -k regex:fused_sweep -s 2 -c 1 -o gpurun_out/prof_fused -f python bench.py --fused --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_fused.log 2>&1; echo "ncu fused rc=$?"
