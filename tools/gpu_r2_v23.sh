cd $GRAFT_REPO_ROOT
BENCH_ARGS="--lmhead --update --steps 5 --warmup 3 --no-unfused --no-e2e --no-cpu" bash tools/gpu_ab.sh dz23 build_variants/lib_cur.so build_variants/lib_dz256.so
