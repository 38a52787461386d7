timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_lmhead_update_gpu.py -q -x 2>&1 | tail -3
DART_GEMM_2SM=0 timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x 2>&1 | tail -1
for v in 1 0; do DART_GEMM_2SM=$v timeout 600 python bench.py --lmhead --update --steps 5 --warmup 3 --no-unfused 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read()); print('2sm=$v', j['ms_per_step'], 'ms', round(j['roofline']['achieved'],1), 'TF', j['clocks']['sm_mhz'])"; done
