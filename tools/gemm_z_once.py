import sys
sys.path.insert(0, '.')
import torch
from paper_2509_23866_b200 import dart
dev = torch.device("cuda", 0)
M, d, V = 8192, 3584, 152064
h = (torch.randn(M, d, device=dev) * 0.5).to(torch.bfloat16)
W = (torch.randn(V, d, device=dev) * 0.02).to(torch.bfloat16)
z32 = torch.empty(M, V, device=dev)
torch.cuda.synchronize()
dart.gemm_bf16(h, W, z32)
torch.cuda.synchronize()
