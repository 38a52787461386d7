export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
DART_GEMM_2SM=4 timeout 120 python tools/g2_small.py 2>&1 | tail -3; echo "small rc=$?"
DART_GEMM_2SM=4 timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x 2>&1 | tail -3 | sed 's/^/mc4 gemm /'
timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x 2>&1 | tail -1 | sed 's/^/default gemm /'
if DART_GEMM_2SM=4 timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x > /dev/null 2>&1; then
  DART_GEMM_2SM=4 timeout 300 python -m pytest tests/test_lmhead_update_gpu.py -m gpu -q -x 2>&1 | tail -1 | sed 's/^/mc4 update /'
  for v in 4 1; do for i in 0 3 5; do DART_GEMM_2SM=$v timeout 300 python tools/gemm_power.py $i 2>&1 | grep -E "case|Error" | sed "s/^/2SM=$v /" | head -2; done; done
  for v in 4 1 4 1; do DART_GEMM_2SM=$v timeout 600 python bench.py --lmhead --update --steps 5 --warmup 3 --no-unfused > gpurun_out/bench_lmup_mc.json 2>/dev/null; python -c "
import json; j=json.load(open('gpurun_out/bench_lmup_mc.json')); print('2SM=$v', j['ms_per_step'], round(j['roofline']['achieved']), j['clocks'])"; done
fi
