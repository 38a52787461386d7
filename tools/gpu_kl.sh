mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_kl_gpu.py -q --timeout 900 > gpurun_out/pytest_kl.log 2>&1; echo "kl pytest rc=$?"; tail -4 gpurun_out/pytest_kl.log
