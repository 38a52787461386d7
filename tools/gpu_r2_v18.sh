cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_fused_gpu.py tests/test_curation.py -q -x -m gpu > gpurun_out/r2v18_tests.log 2>&1; tail -1 gpurun_out/r2v18_tests.log
timeout 900 compute-sanitizer --tool initcheck --kernel-regex kns=dart --error-exitcode 9 python tools/sanitize_driver.py lmhead lmupdate fused klexact > gpurun_out/r02_sanitize_initcheck_dart.log 2>&1; echo "initcheck(dart kernels) rc=$?"; tail -2 gpurun_out/r02_sanitize_initcheck_dart.log
timeout 600 python bench.py --kl exact --steps 20 --warmup 5 > gpurun_out/r02_bench_kl_exact.json 2> gpurun_out/r02_bench_kl_exact.err; tail -c 300 gpurun_out/r02_bench_kl_exact.json
