"""Sustained-loop comparison of the tcgen05 GEMM (dart_gemm_bf16) and cuBLAS
(torch.matmul) on the LM-head update shapes (one 8192-row chunk, d = 3584,
V = 152064): ms per call, TFLOP/s, SM clock and power during the loop."""
import sys, time, json
sys.path.insert(0, '.')
import torch
from paper_2509_23866_b200 import dart
import bench

dev = torch.device("cuda", 0)
M, d, V = 8192, 3584, 152064
g = torch.Generator(device=dev).manual_seed(0)
h = (torch.randn(M, d, device=dev, generator=g) * 0.5).to(torch.bfloat16)
W = (torch.randn(V, d, device=dev, generator=g) * 0.02).to(torch.bfloat16)
dz = (torch.randn(M, V, device=dev, generator=g) * 1e-4).to(torch.bfloat16)
z32 = torch.empty(M, V, device=dev)
zb = torch.empty(M, V, device=dev, dtype=torch.bfloat16)
dh32 = torch.empty(M, d, device=dev)
dhb = torch.empty(M, d, device=dev, dtype=torch.bfloat16)
dW32 = torch.zeros(V, d, device=dev)
dWb = torch.empty(V, d, device=dev, dtype=torch.bfloat16)
fl = 2.0 * M * d * V

cases = {
    "ours z (fp32 out)": lambda: dart.gemm_bf16(h, W, z32),
    "ours z (bf16 out)": lambda: dart.gemm_bf16(h, W, zb),
    "cublas z (bf16 out)": lambda: torch.matmul(h, W.t(), out=zb),
    "ours dh (fp32 out)": lambda: dart.gemm_bf16(dz, W, dh32, b_mn_major=True),
    "cublas dh (bf16 out)": lambda: torch.matmul(dz, W, out=dhb),
    "ours dW (fp32 accumulate)": lambda: dart.gemm_bf16(dz, h, dW32, a_mn_major=True, b_mn_major=True,
                                                        mode=dart.GEMM_ACCUM_F32),
    "ours dW (fp32 store)": lambda: dart.gemm_bf16(dz, h, dW32, a_mn_major=True, b_mn_major=True,
                                                   mode=dart.GEMM_STORE_F32),
    "cublas dW (bf16 out)": lambda: torch.matmul(dz.t(), h, out=dWb),
}
only = sys.argv[1:] and int(sys.argv[1])
for ci, (name, f) in enumerate(cases.items()):
    if only is not False and only != "" and sys.argv[1:] and ci != only:
        continue
    print("running", name, flush=True)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    time.sleep(0.5)
    clk = bench.ClockSampler(0); clk.start(); time.sleep(0.1)
    n = 0
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    t0 = time.time()
    while time.time() - t0 < 1.5:
        for _ in range(20):
            f()
        n += 20
        torch.cuda.synchronize()
    e.record(); torch.cuda.synchronize()
    c = clk.stop() or {}
    ms = s.elapsed_time(e) / n
    print(json.dumps({"case": name, "ms": round(ms, 3), "TFLOPs": round(fl / ms / 1e9, 1), "sm_mhz": c.get("sm_mhz"),
                      "power_w": c.get("power_w")}), flush=True)
