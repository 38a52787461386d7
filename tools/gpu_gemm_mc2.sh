export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_lmhead_update_gpu.py -m gpu -q -x 2>&1 | tail -1 | sed 's/^/default /'
for v in default 4 1 default 4 1; do
  if [ $v = default ]; then unset DART_GEMM_2SM; else export DART_GEMM_2SM=$v; fi
  timeout 600 python bench.py --lmhead --update --steps 5 --warmup 3 --no-unfused > gpurun_out/bench_lmup_mc2.json 2>/dev/null; python -c "
import json; j=json.load(open('gpurun_out/bench_lmup_mc2.json')); print('2SM=$v', j['ms_per_step'], round(j['roofline']['achieved']), j['clocks']['sm_mhz'])"
done
unset DART_GEMM_2SM
timeout 600 python bench.py --lmhead --update --steps 5 --warmup 3 > gpurun_out/bench_lmup_final.json 2>/dev/null; python -c "
import json; j=json.load(open('gpurun_out/bench_lmup_final.json')); print('final', j['ms_per_step'], 'cublas', j['unfused_cublas_pipeline']['ms_per_step'], j['clocks'])"
