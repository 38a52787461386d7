for f in build_variants/*.so; do
  DART_LIB_PATH=$PWD/$f TAG=$f timeout 300 python tools/time_fused.py 2>&1 | tail -1
  DART_LIB_PATH=$PWD/$f TAG=$f timeout 300 python tools/time_fused.py 2>&1 | tail -1
done
