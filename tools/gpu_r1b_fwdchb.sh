export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
DART_LIB_PATH=$PWD/build_variants/f8w8s3.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x 2>&1 | tail -1 | sed 's/^/f8w8s3 parity /'
for f in paper_2509_23866_b200/libdart_loss.so build_variants/f8w8s3.so build_variants/f8w4s3.so build_variants/f8w6s2.so paper_2509_23866_b200/libdart_loss.so build_variants/f8w8s3.so; do echo "== $f"; DART_LIB_PATH=$PWD/$f timeout 600 python tools/diag_loop.py 2>&1 | grep -E '"mode"' | python -c "
import sys,json
for l in sys.stdin:
    j=json.loads(l); c=j['clocks'] or {}
    if j['mode']=='bwd': continue
    print(j['mode'], j['gap'], 'fwd', j['fwd_ms'], j['fwd_frac'], 'bwd', j['bwd_ms'], c.get('sm_mhz'), c.get('power_w'))"; done
