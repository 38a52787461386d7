cd $GRAFT_REPO_ROOT
nproc > gpurun_out/r2_nproc.txt; free -g >> gpurun_out/r2_nproc.txt; lscpu | grep "Model name" >> gpurun_out/r2_nproc.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -s -k "multi_gpu or full_size_vs_oracle or stream_gpu or virtual_ranks" > gpurun_out/r2_t1.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err
