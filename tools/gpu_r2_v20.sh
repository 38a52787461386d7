cd $GRAFT_REPO_ROOT
bash tools/gpu_ab.sh bwd20 build_variants/lib_cur.so build_variants/lib_bwds3.so build_variants/lib_bwds5.so build_variants/lib_bwds6.so build_variants/lib_bwd16w2k.so build_variants/lib_bwd16w2k6.so build_variants/lib_bwd12w2k6.so
