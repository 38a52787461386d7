# ncu --set full of the two LM-head kernels (forward and dz epilogue) at the single config
# (outputs gpurun_out/prof_lmfwd.ncu-rep, prof_lmdz.ncu-rep); then, here: python tools/summarize_profiles.py <tag>
cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:lmhead_kernel<\(bool\)0>' -s 1 -c 1 -o gpurun_out/prof_lmfwd -f python bench.py --lmhead --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_lmfwd.log 2>&1; echo "ncu lmfwd rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:lmhead_kernel<\(bool\)1>' -s 1 -c 1 -o gpurun_out/prof_lmdz -f python bench.py --lmhead --update --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_lmdz.log 2>&1; echo "ncu lmdz rc=$?"
