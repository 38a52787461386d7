cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_fused_gpu.py -q -x > gpurun_out/r2v5_fused_tests.log 2>&1
tail -2 gpurun_out/r2v5_fused_tests.log
BENCH_ARGS="--fused --steps 20 --warmup 5 --no-e2e --no-cpu" bash tools/gpu_ab.sh fu5 build_variants/lib_fold.so build_variants/lib_pipe15.so build_variants/lib_pipe16.so
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_driver.py fused > gpurun_out/r2v5_san_$tool.log 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY| ok" gpurun_out/r2v5_san_$tool.log | head -3
done
