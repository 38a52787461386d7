cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
DART_LIB_PATH=$PWD/build_variants/lib_fu_p2ldg.so timeout 900 python -m pytest tests/test_fused_gpu.py -q -x > gpurun_out/r2v15_fused_tests.log 2>&1
tail -1 gpurun_out/r2v15_fused_tests.log
BENCH_ARGS="--fused --steps 20 --warmup 5 --no-e2e --no-cpu" bash tools/gpu_ab.sh fu15 build_variants/lib_fu3_la0.so build_variants/lib_fu_p2ldg.so
DART_LIB_PATH=$PWD/build_variants/lib_fu_p2ldg.so timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:fused_sweep -s 1 -c 1 --csv python bench.py --fused --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2v15_ncu.csv 2>&1
