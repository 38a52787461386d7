"""Exactness + timing of the CTA-pair GEMM (DART_GEMM_2SM=1) vs the 1-SM kernel."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_23866_b200 import dart
from oracle import dart_oracle as O

def ints(shape, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(-3, 4, shape, generator=g).to(torch.bfloat16)

for (M, N, K) in ([] if os.environ.get("NOCHECK") else [(256, 256, 64), (300, 520, 200), (1000, 264, 1032), (4096, 2048, 512)]):
    A, B = ints((M, K), 1), ints((N, K), 2)
    ref = O.lmhead_logits(A.float().numpy(), B.float().numpy())
    C = torch.full((M, N), float("nan"), device="cuda")
    dart.gemm_bf16(A.cuda(), B.cuda(), C)
    torch.cuda.synchronize()
    ok = np.array_equal(C.cpu().numpy().astype(np.float64), ref)
    dart.gemm_bf16(A.cuda(), B.cuda(), C, mode=dart.GEMM_ACCUM_F32)
    torch.cuda.synchronize()
    ok2 = np.array_equal(C.cpu().numpy().astype(np.float64), 2 * ref)
    print(f"M={M} N={N} K={K} exact={ok} accum={ok2}", flush=True)

M, N, K = 8192, 152064, 3584
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
C = torch.empty(M, N, device="cuda")
for _ in range(2):
    dart.gemm_bf16(A, B, C)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = int(os.environ.get("ITERS", "10"))
s.record()
for _ in range(n):
    dart.gemm_bf16(A, B, C)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / n
print(f"{os.environ.get('DART_GEMM_2SM', '0')}: {ms:.3f} ms  {2 * M * N * K / ms / 1e9:.1f} TFLOP/s", flush=True)
