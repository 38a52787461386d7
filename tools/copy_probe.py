"""Probe: what kernel does torch's D2D copy_ (the MEASURED_PEAKS copy peak) run,
and at what rate, for a logits-sized buffer (18.7 GB)?  Run under ncu to see
the kernel's launch configuration and memory metrics."""
import sys
import torch
n = 61440 * 152064
a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
a.fill_(1.0)
b = torch.empty_like(a)
for _ in range(3):
    b.copy_(a)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
k = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for _ in range(k):
    b.copy_(a)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / k
print(f"copy_ {ms:.3f} ms  {2 * a.numel() * 2 / ms / 1e6:.1f} GB/s")
