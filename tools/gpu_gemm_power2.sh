export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for i in 0 1 2; do timeout 300 python tools/gemm_power.py $i 2>&1 | grep -E "case|Error" | head -2; done
for i in 0 1 3; do DART_GEMM_2SM=0 timeout 300 python tools/gemm_power.py $i 2>&1 | grep -E "case|Error" | sed 's/^/1cta /' | head -2; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second --clock-control none --csv python tools/gemm_once.py > gpurun_out/gemm_ncu.csv 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/gemm_ncu.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
d=collections.OrderedDict()
for r in rows[1:]:
    d.setdefault((r[ii], r[ki][:60]), {})[r[mi]]=r[vi]
for k,v in d.items(): print(k, v)
PY
