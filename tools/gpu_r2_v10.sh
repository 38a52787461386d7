cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_fused_gpu.py -q -x > gpurun_out/r2v10_fused_tests.log 2>&1
tail -2 gpurun_out/r2v10_fused_tests.log
BENCH_ARGS="--fused --steps 20 --warmup 5 --no-e2e --no-cpu" bash tools/gpu_ab.sh fu10 build_variants/lib_fold_i32.so build_variants/lib_cur.so
bash tools/gpu_ab.sh bwd10 build_variants/lib_cur.so build_variants/lib_bwd_i32.so
