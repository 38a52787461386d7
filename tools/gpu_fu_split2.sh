for f in build_variants/*.so; do
  for v in 0 2; do
    DART_LIB_PATH=$PWD/$f DART_FUSED_VARIANT=$v TAG="$f v$v" timeout 300 python tools/time_fused.py 2>&1 | tail -1
  done
done
