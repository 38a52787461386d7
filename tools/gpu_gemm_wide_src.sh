export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
DART_GEMM_2SM=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_bf16 -c 1 -o gpurun_out/prof_gemm_wide2 -f python tools/gemm_z_once.py > /dev/null 2>&1; echo "wide rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_bf16 -c 1 -o gpurun_out/prof_gemm_pair2 -f python tools/gemm_z_once.py > /dev/null 2>&1; echo "pair rc=$?"
