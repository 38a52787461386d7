export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  DART_GEMM_2SM=4 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_driver.py lmupdate > gpurun_out/sanitize7_$tool.log 2>&1; echo "mc $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/sanitize7_$tool.log | head -2; grep "Race reported" gpurun_out/sanitize7_$tool.log | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | head -3
done
grep -E "and (Read|Write) access" gpurun_out/sanitize7_racecheck.log | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | head -5
