cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
DART_LIB_PATH=$PWD/build_variants/lib_pipe.so timeout 900 python -m pytest tests/test_fused_gpu.py -q -x > gpurun_out/r2v4_fused_tests.log 2>&1
tail -2 gpurun_out/r2v4_fused_tests.log
BENCH_ARGS="--fused --steps 20 --warmup 5 --no-e2e --no-cpu" bash tools/gpu_ab.sh fu build_variants/lib_fold.so build_variants/lib_pipe.so
for v in lm_base lm_h1 lm_h2 lm_g2 lm_g6 lm_h1g6; do
  DART_LIB_PATH=$PWD/build_variants/$v.so timeout 600 python bench.py --lmhead --no-unfused --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/lm_$v.json 2> gpurun_out/lm_$v.err
  DART_LIB_PATH=$PWD/build_variants/$v.so timeout 600 ncu --metrics dram__bytes_read.sum,lts__t_bytes.sum,gpu__time_duration.sum --clock-control none -k regex:lmhead_kernel -c 1 --csv python bench.py --lmhead --no-unfused --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/lm_ncu_$v.csv 2>&1
done
