cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python -m pytest tests/test_kl_gpu.py -q -x > gpurun_out/r2v17_kl_tests.log 2>&1; tail -1 gpurun_out/r2v17_kl_tests.log
BENCH_ARGS="--kl exact --steps 20 --warmup 5 --no-e2e --no-cpu" bash tools/gpu_ab.sh kl17 build_variants/lib_cur.so build_variants/lib_klfast.so
bash tools/gpu_bench_prof.sh
bash tools/gpu_sanitize.sh r02
