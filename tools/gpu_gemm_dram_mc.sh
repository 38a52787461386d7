export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum --clock-control none --csv -k regex:gemm_bf16 python tools/gemm_once.py > gpurun_out/gemm_ncu_mc.csv 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/gemm_ncu_mc.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
d=collections.OrderedDict()
for r in rows[1:]:
    d.setdefault((r[ii], r[ki][:50]), {})[r[mi]]=r[vi]
for k,v in d.items(): print(k, {m.split('.')[0]: x for m,x in v.items()})
PY
