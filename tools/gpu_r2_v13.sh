cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_fused_gpu.py tests/test_parity_gpu.py -q -x > gpurun_out/r2v13_tests.log 2>&1
tail -2 gpurun_out/r2v13_tests.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_driver.py fused tiny odd > gpurun_out/r2v13_san_$tool.log 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/r2v13_san_$tool.log | head -3
done
bash tools/gpu_ab.sh bwd13 build_variants/lib_cur.so build_variants/lib_bwdlds.so
timeout 600 python bench.py --fused --steps 20 --warmup 5 > gpurun_out/r2v13_fused_bench.json 2> gpurun_out/r2v13_fused_bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_sweep -s 1 -c 1 -o gpurun_out/prof_fused_r2 -f python bench.py --fused --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2v13_ncu.log 2>&1
