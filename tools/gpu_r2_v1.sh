cd $GRAFT_REPO_ROOT
lscpu | grep "Model name" > gpurun_out/r2v1_cpu.txt; nproc >> gpurun_out/r2v1_cpu.txt; nvidia-smi -L >> gpurun_out/r2v1_cpu.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2v1_smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2v1_bench.json 2> gpurun_out/r2v1_bench.err
timeout 900 python bench.py --lmhead --update --steps 5 --warmup 3 > gpurun_out/r2v1_lmupd.json 2> gpurun_out/r2v1_lmupd.err
timeout 600 python bench.py --fused --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/r2v1_fused.json 2> gpurun_out/r2v1_fused.err
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/r2v1_tests.log 2>&1
