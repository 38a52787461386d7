export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for cr in 8192 16384 30720; do
  extra="--no-unfused"; [ $cr = 8192 ] && extra=""
  timeout 900 python bench.py --lmhead --update --chunk-rows $cr --steps 5 --warmup 3 $extra > gpurun_out/bench_lmup_$cr.json 2>gpurun_out/bench_lmup_$cr.err; echo "cr=$cr rc=$?"
  python -c "
import json; j=json.load(open('gpurun_out/bench_lmup_$cr.json')); u=j.get('unfused_cublas_pipeline') or {}; print('chunk', $cr, j['ms_per_step'], round(j['roofline']['achieved']), 'cublas', u.get('ms_per_step'), j['clocks'])"
done
