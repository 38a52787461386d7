cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build3.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/r2_bench3.json 2> gpurun_out/r2_bench3.err
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2_t3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lmhead -c 4 --csv --log-file gpurun_out/r2_lm_launches.csv python bench.py --lmhead --update --steps 1 --warmup 3 --no-unfused > /dev/null 2>&1
