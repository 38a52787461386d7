cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
DART_LIB_PATH=$PWD/build_variants/lib_fufast3.so timeout 900 python -m pytest tests/test_fused_gpu.py -q -x > gpurun_out/r2v11_fused_tests.log 2>&1
tail -2 gpurun_out/r2v11_fused_tests.log
BENCH_ARGS="--fused --steps 20 --warmup 5 --no-e2e --no-cpu" bash tools/gpu_ab.sh fu11 build_variants/lib_cur.so build_variants/lib_fufast1.so build_variants/lib_fufast2.so build_variants/lib_fufast3.so
