cd $GRAFT_REPO_ROOT
free -g > gpurun_out/r2v21_mem.txt; cat /sys/fs/cgroup/memory.max >> gpurun_out/r2v21_mem.txt 2>&1; nproc >> gpurun_out/r2v21_mem.txt; nvidia-smi --query-gpu=name,memory.total,power.limit --format=csv >> gpurun_out/r2v21_mem.txt
bash tools/gpu_ab.sh bwd21 build_variants/lib_cur.so build_variants/lib_bwds5.so
