export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for v in 1 2; do DART_GEMM_2SM=$v timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_lmhead_update_gpu.py -m gpu -q -x 2>&1 | tail -1 | sed "s/^/2SM=$v /"; done
for v in 2 1; do for i in 0 3 5; do DART_GEMM_2SM=$v timeout 300 python tools/gemm_power.py $i 2>&1 | grep -E "case|Error" | sed "s/^/cst 2SM=$v /" | head -2; done; done
for v in 2 1; do DART_GEMM_2SM=$v timeout 600 python bench.py --lmhead --update --steps 5 --warmup 3 --no-unfused > gpurun_out/bench_lmup_c.json 2>/dev/null; python -c "
import json; j=json.load(open('gpurun_out/bench_lmup_c.json')); print('cst 2SM=$v', j['ms_per_step'], round(j['roofline']['achieved']), j['clocks'])"; done
DART_LIB_PATH=$PWD/build_variants/nocst.so DART_GEMM_2SM=1 timeout 600 python bench.py --lmhead --update --steps 5 --warmup 3 > gpurun_out/bench_lmup_nc.json 2>/dev/null; python -c "
import json; j=json.load(open('gpurun_out/bench_lmup_nc.json')); print('nocst 2SM=1', j['ms_per_step'], round(j['roofline']['achieved']), j['clocks'], 'cublas', j['unfused_cublas_pipeline']['ms_per_step'])"
