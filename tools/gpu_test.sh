mkdir -p gpurun_out
timeout 300 python tools/debug_row.py > gpurun_out/debug_row.log 2>&1; cat gpurun_out/debug_row.log | tail -15
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 --maxfail 40 > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu4.log
