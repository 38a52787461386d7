cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:lmhead_kernel -s 2 -c 2 -o gpurun_out/prof_lmupd -f python bench.py --lmhead --update --steps 1 --warmup 1 --no-unfused > gpurun_out/r2v22_ncu.log 2>&1; echo "ncu rc=$?"
