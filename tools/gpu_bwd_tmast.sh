export PATH=/usr/local/cuda/bin:$PATH
DART_LIB_PATH=$PWD/build_variants/bwd_tmast.so timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_virtual_ranks.py tests/test_stream_gpu.py -q -x 2>&1 | tail -3
for v in bwd_base bwd_tmast bwd_base bwd_tmast; do
  DART_LIB_PATH=$PWD/build_variants/$v.so timeout 600 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']
print('$v', round(j['value']/1e6,3), 'M tok/s  fwd', round(k['fwd_sweep']['avg_ms'],3), 'bwd', round(k['bwd_sweep']['avg_ms'],3), 'ms', round(k['bwd_sweep']['frac'],3), j['clocks']['sm_mhz'])"
done
DART_LIB_PATH=$PWD/build_variants/bwd_tmast.so timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_driver.py tiny midsplit 2>&1 | grep -E "SUMMARY|ok"
DART_LIB_PATH=$PWD/build_variants/bwd_tmast.so timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_driver.py tiny midsplit odd 2>&1 | grep -E "SUMMARY|ok"
