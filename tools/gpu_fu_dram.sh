export PATH=/usr/local/cuda/bin:$PATH
for f in build_variants/fu_ctas1.so build_variants/fu_ctas1_nc16.so ""; do
  if [ -n "$f" ]; then export DART_LIB_PATH=$PWD/$f; else unset DART_LIB_PATH; fi
  TAG=${f:-default} timeout 300 python tools/time_fused.py 2>&1 | tail -1
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:fused_sweep -s 3 -c 1 python tools/time_fused.py 2>&1 | grep -E "dram__bytes|gpu__time|hit_rate"
done
