mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_gpu_t2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_t2.log
bash tools/gpu_tune.sh
