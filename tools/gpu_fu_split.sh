export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python -m pytest tests/test_fused_gpu.py -q -x 2>&1 | tail -3
for v in 0 2; do
  DART_FUSED_VARIANT=$v TAG=variant$v timeout 300 python tools/time_fused.py 2>&1 | tail -1
  DART_FUSED_VARIANT=$v TAG=variant$v timeout 300 python tools/time_fused.py 2>&1 | tail -1
  DART_FUSED_VARIANT=$v timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fused_sweep -s 3 -c 1 python tools/time_fused.py 2>&1 | grep -E "dram__bytes|gpu__time"
done
