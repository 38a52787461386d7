# Round-2 final evidence: every bench line + GPU suite + smoke (outputs gpurun_out/r02f_*)
cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; tail -1 gpurun_out/r02f_smoke.log
timeout 900 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02f_bench_reference.json 2> gpurun_out/r02f_bench_reference.err
timeout 600 python bench.py --fused --steps 20 --warmup 5 > gpurun_out/r02f_bench_fused.json 2> gpurun_out/r02f_bench_fused.err
timeout 600 python bench.py --kl exact --steps 20 --warmup 5 --no-e2e > gpurun_out/r02f_bench_kl_exact.json 2> gpurun_out/r02f_bench_kl_exact.err
timeout 900 python bench.py --lmhead --steps 5 --warmup 3 > gpurun_out/r02f_bench_lmhead.json 2> gpurun_out/r02f_bench_lmhead.err
timeout 900 python bench.py --lmhead --update --steps 5 --warmup 3 > gpurun_out/r02f_bench_lmhead_update.json 2> gpurun_out/r02f_bench_lmhead_update.err
for c in long adaptive scale20 scale22 scale24; do
  timeout 1500 python bench.py --config $c --stream-rows 32768 --pool 3 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02f_bench_stream_$c.json 2> gpurun_out/r02f_bench_stream_$c.err
done
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r02f_gpu_tests.log 2>&1; tail -2 gpurun_out/r02f_gpu_tests.log
