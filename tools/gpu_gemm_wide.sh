export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
DART_GEMM_2SM=2 timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x > gpurun_out/pytest_wide.log 2>&1; echo "pytest wide rc=$?"; tail -5 gpurun_out/pytest_wide.log
if grep -q passed gpurun_out/pytest_wide.log && ! grep -q failed gpurun_out/pytest_wide.log; then
DART_GEMM_2SM=2 timeout 300 python -m pytest tests/test_lmhead_update_gpu.py -m gpu -q -x > gpurun_out/pytest_wide2.log 2>&1; echo "pytest wide2 rc=$?"; tail -3 gpurun_out/pytest_wide2.log
for i in 0 3 5; do DART_GEMM_2SM=2 timeout 300 python tools/gemm_power.py $i 2>&1 | grep -E "case|Error" | sed 's/^/wide /' | head -2; done
for i in 0 3 5; do timeout 300 python tools/gemm_power.py $i 2>&1 | grep -E "case|Error" | sed 's/^/pair /' | head -2; done
for v in 2 1 2 1; do DART_GEMM_2SM=$v timeout 600 python bench.py --lmhead --update --steps 5 --warmup 3 --no-unfused > gpurun_out/bench_lmup_w.json 2>/dev/null; python -c "
import json; j=json.load(open('gpurun_out/bench_lmup_w.json')); print('2SM=$v', j['ms_per_step'], round(j['roofline']['achieved']), j['clocks'])"; done
fi
