mkdir -p gpurun_out
for f in build_variants/*.so; do
  DART_LIB_PATH=$PWD/$f timeout 120 python bench.py --fused --steps 10 --warmup 3 --no-cpu --no-e2e 2>gpurun_out/tf_err.log > gpurun_out/tf.json; r=$?
  python -c "
import json,sys; d=json.load(open('gpurun_out/tf.json')); k=d['kernels']
print('$f', round(d['value']/1e6,3),'Mtok/s', 'kernel', round(k['bwd_sweep']['frac'],3), round(k['bwd_sweep']['avg_ms'],3))" 2>/dev/null || echo "$f FAILED rc=$r"
done
timeout 900 python -m pytest tests/test_fused_gpu.py -q 2>&1 | tail -2
