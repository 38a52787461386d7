"""One launch of each LM-head update GEMM (chunk of 8192 rows) for ncu."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2509_23866_b200 import dart
dev = torch.device("cuda", 0)
M, d, V = 8192, 3584, 152064
h = (torch.randn(M, d, device=dev) * 0.5).to(torch.bfloat16)
W = (torch.randn(V, d, device=dev) * 0.02).to(torch.bfloat16)
dz = (torch.randn(M, V, device=dev) * 1e-4).to(torch.bfloat16)
z32 = torch.empty(M, V, device=dev)
zb = torch.empty(M, V, device=dev, dtype=torch.bfloat16)
dh32 = torch.empty(M, d, device=dev)
dW32 = torch.zeros(V, d, device=dev)
dhb = torch.empty(M, d, device=dev, dtype=torch.bfloat16)
dWb = torch.empty(V, d, device=dev, dtype=torch.bfloat16)
torch.cuda.synchronize()
dart.gemm_bf16(h, W, z32)
dart.gemm_bf16(h, W, zb)
dart.gemm_bf16(dz, W, dh32, b_mn_major=True)
dart.gemm_bf16(dz, h, dW32, a_mn_major=True, b_mn_major=True, mode=dart.GEMM_ACCUM_F32)
torch.matmul(h, W.t(), out=zb)
torch.matmul(dz, W, out=dhb)
torch.matmul(dz.t(), h, out=dWb)
torch.cuda.synchronize()
