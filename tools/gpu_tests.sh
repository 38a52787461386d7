mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 --maxfail 20 > gpurun_out/pytest_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu_all.log
