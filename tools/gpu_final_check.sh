export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_driver.py lmhead lmupdate > gpurun_out/sanitize4_$tool.log 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/sanitize4_$tool.log | head -2
done
timeout 900 python bench.py --lmhead --update --steps 5 --warmup 3 > gpurun_out/bench_lmup.json 2>/dev/null; python -c "
import json; j=json.load(open('gpurun_out/bench_lmup.json')); print('update', j['ms_per_step'], j['roofline']['achieved'], j['unfused_cublas_pipeline']['ms_per_step'], j['clocks'])"
