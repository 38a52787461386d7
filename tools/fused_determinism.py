"""Run-to-run determinism of the fused update at the single config (6 runs):
logits untouched, masked rows zero, kept-row lse and the workspace bitwise
equal across runs.  Usage (on the GPU box): python tools/fused_determinism.py"""
import sys
sys.path.insert(0, '.')
import torch, numpy as np
from paper_2509_23866_b200 import dart, synth
from tests.gpu_helpers import run_gpu
b = synth.make_batch("single", seed=0, device="cuda")
cfg = dart.Config()
old = run_gpu(b, cfg)
keep, norm = old.keep.clone(), old.norm.clone()
del old
dev = torch.device("cuda")
ck0 = b.logits.view(torch.int16).sum(dtype=torch.int64).item()
kt = torch.repeat_interleave(keep[:b.layout.S].bool(), torch.as_tensor(np.diff(b.layout.step_tok_off), device=dev))
ref = None
for it in range(6):
    dl = dart.DartLoss(b.layout, dart.whole_shard(b.layout), b.V, cfg, dev)
    dl.ws.fill_(0)
    dl.fused(b.logits, b.target, b.logp_old, b.logp_rollout, b.logp_ref, keep=keep, norm=norm)
    torch.cuda.synchronize()
    ck = b.logits.view(torch.int16).sum(dtype=torch.int64).item()
    masked_nz = int(torch.count_nonzero(dl.dlogits[~kt]))
    cur = (dl.lse.clone(), dl.ws.clone())
    if ref is None:
        ref = cur
    dlse = int(((cur[0] != ref[0]) & kt).sum())
    dws = torch.nonzero(cur[1] != ref[1])[:, 0]
    print(it, "logits checksum same:", ck == ck0, "masked nonzero:", masked_nz, "lse rows differ:", dlse,
          "ws bytes differ:", dws.numel(), "ws first diff offsets:", dws[:6].tolist(), "ws bytes", dl.ws_bytes, flush=True)
    del dl
