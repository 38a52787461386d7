"""Time dart_loss_fused alone on the single config (no status check: for
timing experiments with DART_FC_EXP variants).  Prints ms and M tokens/s."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_23866_b200 import dart, synth  # noqa: E402

b = synth.make_batch("single", device="cuda")
cfg = dart.Config()
dl = dart.DartLoss(b.layout, dart.whole_shard(b.layout), b.V, cfg, "cuda")
args = (b.logits, b.target, b.logp_old, b.logp_rollout, b.logp_ref)
dl.run(*args)
torch.cuda.synchronize()
keep, norm = dl.keep.clone(), dl.norm.clone()
for _ in range(3):
    dl.fused(*args, keep=keep, norm=norm)
torch.cuda.synchronize()
n = int(os.environ.get("STEPS", "20"))
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(n):
    dl.fused(*args, keep=keep, norm=norm)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / n
print(f"{os.environ.get('TAG', '')} {ms:.3f} ms  {b.layout.T / ms / 1e3:.3f} M tok/s", flush=True)
