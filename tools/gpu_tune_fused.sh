mkdir -p gpurun_out
for f in build_variants/*.so; do
  DART_LIB_PATH=$PWD/$f timeout 300 python bench.py --fused --steps 20 --warmup 3 --no-cpu --no-e2e 2>gpurun_out/tf_err.log > gpurun_out/tf.json; tail -2 gpurun_out/tf_err.log; cat gpurun_out/tf.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('$f', round(d['value']/1e6,3),'Mtok/s', 'kernel', round(k['bwd_sweep']['frac'],3), round(k['bwd_sweep']['avg_ms'],3), d['clocks']['sm_mhz'])"
done
