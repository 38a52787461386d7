export PATH=/usr/local/cuda/bin:$PATH
for f in build_variants/prev.so paper_2509_23866_b200/libdart_loss.so build_variants/prev.so paper_2509_23866_b200/libdart_loss.so; do echo "== $f"; DART_LIB_PATH=$PWD/$f timeout 600 python tools/diag_loop.py 2>&1 | grep -E '"mode"' | python -c "
import sys,json
for l in sys.stdin:
    j=json.loads(l); c=j['clocks'] or {}
    if j['mode']=='fwd': continue
    print(j['mode'], j['gap'], 'fwd', j['fwd_ms'], 'bwd', j['bwd_ms'], j['bwd_frac'], c.get('sm_mhz'), c.get('power_w'))"; done
nvidia-smi --query-gpu=name,memory.total,clocks.max.mem,power.limit,vbios_version --format=csv
