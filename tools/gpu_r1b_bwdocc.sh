export PATH=/usr/local/cuda/bin:$PATH
for f in paper_2509_23866_b200/libdart_loss.so build_variants/w12s4.so build_variants/w16s3.so build_variants/w6s4m2.so build_variants/w8s3m2.so paper_2509_23866_b200/libdart_loss.so; do echo "== $f"; DART_LIB_PATH=$PWD/$f timeout 600 python tools/diag_loop.py 2>&1 | grep -E '"mode"' | python -c "
import sys,json
for l in sys.stdin:
    j=json.loads(l); c=j['clocks'] or {}
    if j['mode']=='fwd': continue
    print(j['mode'], j['gap'], 'fwd', j['fwd_ms'], 'bwd', j['bwd_ms'], j['bwd_frac'], c.get('sm_mhz'), c.get('power_w'))"; done
