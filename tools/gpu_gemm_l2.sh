export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
M=lts__t_bytes.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_requests_op_read.sum,lts__t_requests_op_write.sum,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcunit_ltcfabric.sum,lts__t_sectors_lookup_hit.sum,lts__t_sectors_lookup_miss.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__m_xbar2l1tex_read_bytes.sum,l1tex__m_l1tex2xbar_write_bytes.sum
timeout 600 ncu --metrics $M --clock-control none --csv -k regex:"gemm|nvjet" python tools/gemm_once2.py > gpurun_out/gemm_l2.csv 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/gemm_l2.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
d=collections.OrderedDict()
for r in rows[1:]:
    d.setdefault((r[ii], r[ki][:40]), {})[r[mi]]=r[vi]
for k,v in d.items():
    print(k)
    for m,x in v.items(): print('   ', m, x)
PY
