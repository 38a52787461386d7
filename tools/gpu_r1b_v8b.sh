export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for f in build_variants/v8i.so build_variants/old.so build_variants/full2.so build_variants/v8iw12.so build_variants/v8i.so build_variants/old.so; do echo "== $f"; DART_LIB_PATH=$PWD/$f timeout 600 python tools/diag_loop.py 2>&1 | grep -E '"mode"' | python -c "
import sys,json
for l in sys.stdin:
    j=json.loads(l); c=j['clocks'] or {}
    print(j['mode'], j['gap'], 'fwd', j['fwd_ms'], j['fwd_frac'], 'bwd', j['bwd_ms'], j['bwd_frac'], c.get('sm_mhz'), c.get('power_w'))"; done
DART_LIB_PATH=$PWD/build_variants/v8i.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_sweep -s 2 -c 1 -o gpurun_out/prof_bwd_v8i -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_bwd_v8i.log 2>&1; echo "ncu rc=$?"
