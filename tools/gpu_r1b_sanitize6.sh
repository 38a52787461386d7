export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_driver.py tiny small_multi odd midsplit fused klexact > gpurun_out/sanitize6_$tool.log 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/sanitize6_$tool.log | head -2
done
