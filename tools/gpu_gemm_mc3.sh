export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
DART_GEMM_2SM=5 timeout 120 python tools/g2_small.py 2>&1 | tail -3
DART_GEMM_2SM=5 timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_lmhead_update_gpu.py -m gpu -q -x 2>&1 | tail -1 | sed 's/^/mc5 /'
for v in 5 1 5 1; do DART_GEMM_2SM=$v timeout 300 python tools/gemm_power.py 0 2>&1 | grep -E "case|Error" | sed "s/^/2SM=$v /" | head -2; done
for v in 5 4; do DART_GEMM_2SM=$v timeout 300 python tools/gemm_power.py 3 2>&1 | grep -E "case|Error" | sed "s/^/2SM=$v /" | head -2; DART_GEMM_2SM=$v timeout 300 python tools/gemm_power.py 5 2>&1 | grep -E "case|Error" | sed "s/^/2SM=$v /" | head -2; done
