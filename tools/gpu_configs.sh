mkdir -p gpurun_out
for cfg in long adaptive scale20 scale22 scale24; do
  timeout 900 python bench.py --config $cfg --stream-rows 32768 --pool 3 --steps 3 --warmup 3 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; echo "$cfg rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_$cfg.json')); print('$cfg', d['config']['global_tokens'], round(d['value']/1e6,3), 'Mtok/s', round(d['roofline']['frac'],3), 'kept', round(d['config']['kept_token_frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/bench_$cfg.err
done
