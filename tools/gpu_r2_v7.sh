cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
DART_LIB_PATH=$PWD/build_variants/lib_pipe15.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_pipe -s 1 -c 1 -o gpurun_out/prof_pipe15 -f python bench.py --fused --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2v7_ncu_pipe.log 2>&1
DART_LIB_PATH=$PWD/build_variants/lib_fold.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_sweep -s 1 -c 1 -o gpurun_out/prof_fold -f python bench.py --fused --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2v7_ncu_fold.log 2>&1
ls -la gpurun_out/*.ncu-rep
