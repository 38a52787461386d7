import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_23866_b200 import dart
for (M, N, K) in [(64, 2048, 64), (960, 3000 // 8 * 8, 256)]:
    A = torch.randint(-3, 4, (M, K)).to(torch.bfloat16).cuda()
    B = torch.randint(-3, 4, (N, K)).to(torch.bfloat16).cuda()
    C = torch.empty(M, N, device="cuda")
    dart.gemm_bf16(A, B, C)
    torch.cuda.synchronize()
    print(M, N, K, torch.equal(C.cpu(), (A.float() @ B.float().T).cpu()), flush=True)
