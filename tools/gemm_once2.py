"""z = h W^T (bf16 out) once with ours and once with cuBLAS, for ncu."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2509_23866_b200 import dart
dev = torch.device("cuda", 0)
M, d, V = 8192, 3584, 152064
h = (torch.randn(M, d, device=dev) * 0.5).to(torch.bfloat16)
W = (torch.randn(V, d, device=dev) * 0.02).to(torch.bfloat16)
zb = torch.empty(M, V, device=dev, dtype=torch.bfloat16)
torch.cuda.synchronize()
dart.gemm_bf16(h, W, zb)
torch.matmul(h, W.t(), out=zb)
torch.cuda.synchronize()
