export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
DART_LIB_PATH=$PWD/build_variants/c8s3.so timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_virtual_ranks.py tests/test_stream_gpu.py -m gpu -q -x 2>&1 | tail -1 | sed 's/^/c8s3 /'
for f in paper_2509_23866_b200/libdart_loss.so build_variants/c8s3.so build_variants/c8s2.so build_variants/c2s8.so paper_2509_23866_b200/libdart_loss.so build_variants/c8s3.so; do echo "== $f"; DART_LIB_PATH=$PWD/$f timeout 600 python tools/diag_loop.py 2>&1 | grep -E '"mode"' | python -c "
import sys,json
for l in sys.stdin:
    j=json.loads(l); c=j['clocks'] or {}
    if j['mode']=='fwd': continue
    print(j['mode'], j['gap'], 'fwd', j['fwd_ms'], 'bwd', j['bwd_ms'], j['bwd_frac'], c.get('sm_mhz'), c.get('power_w'))"; done
