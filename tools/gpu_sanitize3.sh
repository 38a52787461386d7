export PATH=/usr/local/cuda/bin:$PATH
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_driver.py fused > gpurun_out/sanitize3_$tool.log 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/sanitize3_$tool.log | head -3
done
timeout 900 python -m pytest tests/test_fused_gpu.py tests/test_lmhead_update_gpu.py -q 2>&1 | tail -2
timeout 600 python bench.py --fused --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_fused.json 2>/dev/null; cat gpurun_out/bench_fused.json
