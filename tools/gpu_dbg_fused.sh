mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
for tool in synccheck racecheck; do
DART_LIB_PATH=$PWD/build_variants/lib_fu8x24x2.so timeout 1200 compute-sanitizer --tool $tool --print-limit 5 python bench.py --fused --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/dbg_fused_$tool.log 2>&1; echo $tool rc=$?; grep -v "^\s*$" gpurun_out/dbg_fused_$tool.log | grep -v metric | head -20
done
DART_LIB_PATH=$PWD/build_variants/lib_fu8x24x2.so CUDA_LAUNCH_BLOCKING=1 timeout 300 python bench.py --fused --steps 3 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "Error|error|line" | head
