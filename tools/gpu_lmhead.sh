# NEXT #3: LM-head-fused forward -- bench line + one full ncu capture of the tcgen05 kernel
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python bench.py --lmhead --steps ${STEPS:-10} --warmup 3 > gpurun_out/bench_lmhead.json 2> gpurun_out/bench_lmhead.err; echo "bench rc=$?"
cat gpurun_out/bench_lmhead.json; tail -3 gpurun_out/bench_lmhead.err
if [ -z "$NO_NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lmhead_fwd -s 3 -c 1 -o gpurun_out/prof_lmhead -f python bench.py --lmhead --steps 1 --warmup 3 --no-cpu --no-e2e --no-unfused > gpurun_out/ncu_lmhead.log 2>&1; echo "ncu rc=$?"
tail -5 gpurun_out/ncu_lmhead.log
fi
