cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
for v in la1 la2 la0; do
DART_LIB_PATH=$PWD/build_variants/lib_fu3_$v.so timeout 900 python -m pytest tests/test_fused_gpu.py -q -x > gpurun_out/r2v14_fused_tests_$v.log 2>&1
tail -1 gpurun_out/r2v14_fused_tests_$v.log
done
DART_LIB_PATH=$PWD/build_variants/lib_fu3_la1.so timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_driver.py fused odd > gpurun_out/r2v14_san_racecheck.log 2>&1; echo "racecheck rc=$?"; grep -E "RACECHECK SUMMARY" gpurun_out/r2v14_san_racecheck.log
DART_LIB_PATH=$PWD/build_variants/lib_fu3_la1.so timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_driver.py fused odd > gpurun_out/r2v14_san_synccheck.log 2>&1; echo "synccheck rc=$?"; grep -E "ERROR SUMMARY" gpurun_out/r2v14_san_synccheck.log
BENCH_ARGS="--fused --steps 20 --warmup 5 --no-e2e --no-cpu" bash tools/gpu_ab.sh fu14 build_variants/lib_cur.so build_variants/lib_fu3_la1.so build_variants/lib_fu3_la2.so build_variants/lib_fu3_la0.so
