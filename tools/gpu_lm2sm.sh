timeout 600 python -m pytest tests/test_lmhead_gpu.py tests/test_lmhead_update_gpu.py -q -x 2>&1 | tail -3
for v in 1 0 1 0; do DART_LMHEAD_2SM=$v timeout 600 python bench.py --lmhead --steps 10 --warmup 3 --no-unfused --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']; print('2sm=$v', round(j['ms_per_step'],2), 'ms', round(r['achieved'],1), 'TF', round(r['frac'],3), j['clocks']['sm_mhz'])"; done
