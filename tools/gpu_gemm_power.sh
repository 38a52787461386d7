for i in 0 1 2 3 4 5 6 7; do CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/gemm_power.py $i 2>&1 | grep -E "running|case|Error|error" | head -3; done
