cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests/test_lmhead_gpu.py tests/test_lmhead_update_gpu.py -q -x > gpurun_out/r2v6_lm_tests.log 2>&1
tail -2 gpurun_out/r2v6_lm_tests.log
for rep in 1 2; do
for v in lm_r0 lm_r1; do
  DART_LIB_PATH=$PWD/build_variants/$v.so timeout 600 python bench.py --lmhead --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/lm6_${v}_$rep.json 2> gpurun_out/lm6_${v}_$rep.err
done; done
for v in lm_r0 lm_r1; do
  DART_LIB_PATH=$PWD/build_variants/$v.so timeout 600 ncu --metrics dram__bytes_read.sum,lts__t_bytes.sum,gpu__time_duration.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:lmhead_kernel -c 1 --csv python bench.py --lmhead --no-unfused --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/lm6_ncu_$v.csv 2>&1
done
