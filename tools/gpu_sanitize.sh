# compute-sanitizer over the product kernels: tools/gpu_sanitize.sh [tag] [configs...]
# (defaults: every kernel family). Logs: gpurun_out/sanitize_<tag>_<tool>.log
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
tag=${1:-all}; shift
cfgs=${@:-tiny small_multi odd midsplit fused klexact lmhead lmupdate}
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_driver.py $cfgs > gpurun_out/sanitize_${tag}_$tool.log 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|rror| ok" gpurun_out/sanitize_${tag}_$tool.log | head -12
done
