cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_lmhead_gpu.py tests/test_lmhead_update_gpu.py -q -x > gpurun_out/r2v24_lm_tests.log 2>&1; tail -1 gpurun_out/r2v24_lm_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --lmhead --update --steps 5 --warmup 3 > gpurun_out/r02_bench_lmhead_update.json 2> gpurun_out/r02_bench_lmhead_update.err
