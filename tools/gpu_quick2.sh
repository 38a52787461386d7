mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_gpu_q2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_q2.log
timeout 900 python tools/diag_loop.py 2>&1 | tail -6
for i in 1 2; do timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print(round(d['value']/1e6,3),'Mtok/s', 'fwd', round(k['fwd_sweep']['frac'],3), round(k['fwd_sweep']['avg_ms'],3), 'bwd', round(k['bwd_sweep']['frac'],3), round(k['bwd_sweep']['avg_ms'],3), 'step', round(k['step_frac'],3), d['clocks'])"; done
