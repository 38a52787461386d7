cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_fused_gpu.py -q -x > gpurun_out/r2v16_fused_tests.log 2>&1
tail -1 gpurun_out/r2v16_fused_tests.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_driver.py fused odd > gpurun_out/r2v16_san_$tool.log 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/r2v16_san_$tool.log | head -2
done
DART_LIB_PATH=$PWD/build_variants/lib_bwdg2.so timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "not full_size" > gpurun_out/r2v16_bwdg2_tests.log 2>&1
tail -1 gpurun_out/r2v16_bwdg2_tests.log
bash tools/gpu_ab.sh bwd16 build_variants/lib_cur.so build_variants/lib_bwdg2.so build_variants/lib_bwdg4.so
BENCH_ARGS="--fused --steps 20 --warmup 5 --no-e2e --no-cpu" bash tools/gpu_ab.sh fu16 build_variants/lib_cur.so
