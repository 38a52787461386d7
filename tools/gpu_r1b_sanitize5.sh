export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_driver.py lmupdate > gpurun_out/sanitize5_$tool.log 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Race reported|hazard" gpurun_out/sanitize5_$tool.log | sort | uniq -c | head -5
  DART_GEMM_2SM=2 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_driver.py lmupdate > gpurun_out/sanitize5w_$tool.log 2>&1; echo "wide $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Race reported|hazard" gpurun_out/sanitize5w_$tool.log | sort | uniq -c | head -5
done
timeout 600 python bench.py --lmhead --update --steps 5 --warmup 3 > gpurun_out/bench_lmhead_update_s2.json 2>/dev/null; python -c "
import json; j=json.load(open('gpurun_out/bench_lmhead_update_s2.json')); print(j['ms_per_step'], j['roofline']['achieved'], j['unfused_cublas_pipeline']['ms_per_step'], j['clocks'])"
