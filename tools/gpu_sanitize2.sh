mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_driver.py lmhead fused fused_cluster klexact > gpurun_out/sanitize2_$tool.log 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|rror|ok" gpurun_out/sanitize2_$tool.log | head -8
done
