mkdir -p gpurun_out
for f in build_variants/*.so; do
  DART_LIB_PATH=$PWD/$f timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e 2>/dev/null > gpurun_out/tune_$(basename $f .so).json
  python -c "
import json,sys; d=json.load(open('gpurun_out/tune_$(basename $f .so).json')); k=d['kernels']
print('$f', round(d['value']/1e6,3),'Mtok/s', 'fwd', round(k['fwd_sweep']['frac'],3), 'bwd', round(k['bwd_sweep']['frac'],3), 'step', round(k['step_frac'],3), d['clocks'])"
done
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 --maxfail 40 > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu3.log
