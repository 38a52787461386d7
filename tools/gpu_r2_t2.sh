cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2_smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -s -x -k "lmhead or fused or multi_gpu or stream_gpu or abi" > gpurun_out/r2_t2.log 2>&1
timeout 900 python bench.py --lmhead --update --steps 5 --warmup 3 > gpurun_out/r2_lmupd.json 2> gpurun_out/r2_lmupd.err
timeout 600 python bench.py --fused --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/r2_fused.json 2> gpurun_out/r2_fused.err
