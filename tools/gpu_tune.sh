mkdir -p gpurun_out
for rep in 1 2; do
for f in build_variants/*.so; do
  DART_LIB_PATH=$PWD/$f timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e 2>gpurun_out/tune_err.log > gpurun_out/tune_$(basename $f .so).json
  python -c "
import json,sys; d=json.load(open('gpurun_out/tune_$(basename $f .so).json')); k=d['kernels']
print('$f', round(d['value']/1e6,3),'Mtok/s', 'fwd', round(k['fwd_sweep']['frac'],3), 'bwd', round(k['bwd_sweep']['frac'],3), 'step', round(k['step_frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/tune_err.log
done
done
