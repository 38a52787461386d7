# A/B timing of library builds on one box: tools/gpu_ab.sh tag lib1 lib2 ... (bench.py args via BENCH_ARGS)
cd $GRAFT_REPO_ROOT
tag=$1; shift
args=${BENCH_ARGS:---steps 20 --warmup 5 --no-e2e --no-cpu}
for rep in 1 2; do
  for lib in "$@"; do
    n=$(basename $lib .so)
    DART_LIB_PATH=$PWD/$lib timeout 600 python bench.py $args > gpurun_out/ab_${tag}_${n}_$rep.json 2> gpurun_out/ab_${tag}_${n}_$rep.err
  done
done
