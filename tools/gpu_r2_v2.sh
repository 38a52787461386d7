cd $GRAFT_REPO_ROOT
bash tools/gpu_ab.sh bwd build_variants/lib_head.so build_variants/lib_shape1.so
timeout 900 python -m pytest tests/test_multi_gpu.py -q -x > gpurun_out/r2v2_mg.log 2>&1
