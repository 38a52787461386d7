export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_lmhead_update_gpu.py -m gpu -q -x > gpurun_out/pytest_gemm.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gemm.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv -k regex:gemm_bf16 python tools/gemm_once.py > gpurun_out/gemm_ncu2.csv 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/gemm_ncu2.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
d=collections.OrderedDict()
for r in rows[1:]:
    d.setdefault((r[ii], r[ki][:45]), {})[r[mi]]=r[vi]
for k,v in d.items(): print(k, v)
PY
for lib in paper_2509_23866_b200/libdart_loss.so build_variants/nonarrow.so paper_2509_23866_b200/libdart_loss.so; do
DART_LIB_PATH=$PWD/$lib timeout 900 python bench.py --lmhead --update --steps 5 --warmup 3 --no-unfused > gpurun_out/bench_lmup_r.json 2>/dev/null; python -c "
import json; j=json.load(open('gpurun_out/bench_lmup_r.json')); print('$lib', j['ms_per_step'], round(j['roofline']['achieved']), j['clocks'])"
done
