mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python bench.py --kl exact --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_kl.json 2> gpurun_out/bench_kl.err; echo "kl bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_kl.json')); k=d['kernels']
print('exact KL', round(d['value']/1e6,3),'Mtok/s fwd', round(k['fwd_sweep']['frac'],3), round(k['fwd_sweep']['avg_ms'],3), 'bwd', round(k['bwd_sweep']['frac'],3), round(k['bwd_sweep']['avg_ms'],3), 'step', round(k['step_frac'],3))" || tail -5 gpurun_out/bench_kl.err
timeout 900 ncu --set full --clock-control none -k regex:"fwd_kl|bwd_kl" -s 2 -c 2 -o gpurun_out/prof_kl -f python bench.py --kl exact --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_kl.log 2>&1; echo "ncu kl rc=$?"
