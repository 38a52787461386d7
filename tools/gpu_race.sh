export PATH=/usr/local/cuda/bin:$PATH
for cfg in "0 default" "2 default" "0 sw3" "2 sw3"; do
  set -- $cfg
  if [ "$2" = "sw3" ]; then export DART_LIB_PATH=$PWD/build_variants/fu_sw3.so; else unset DART_LIB_PATH; fi
  DART_FUSED_VARIANT=$1 timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_driver.py fused > gpurun_out/race_$1_$2.log 2>&1
  echo "variant $1 $2:"; grep -E "RACECHECK SUMMARY" gpurun_out/race_$1_$2.log
done
