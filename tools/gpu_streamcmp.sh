for r in 61440 32768 16384 8192; do
  timeout 900 python bench.py --config single --stream-rows $r --pool 3 --steps 20 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('rows $r chunks', d['config']['chunks'], round(d['value']/1e6,3), 'Mtok/s', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('resident', round(d['value']/1e6,3), round(d['kernels']['step_frac'],3), d['clocks']['sm_mhz'])"
