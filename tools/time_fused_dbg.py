"""Phase timing of the cluster fused kernel (build with -DDART_FC_EXP=5)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
dbg = torch.zeros(16, dtype=torch.int64, device="cuda")
os.environ["DART_FC_DBG"] = str(dbg.data_ptr())
from paper_2509_23866_b200 import dart, synth  # noqa: E402
b = synth.make_batch("single", device="cuda")
dl = dart.DartLoss(b.layout, dart.whole_shard(b.layout), b.V, dart.Config(), "cuda")
args = (b.logits, b.target, b.logp_old, b.logp_rollout, b.logp_ref)
dl.run(*args)
torch.cuda.synchronize()
keep, norm = dl.keep.clone(), dl.norm.clone()
dl.fused(*args, keep=keep, norm=norm)
torch.cuda.synchronize()
dbg.zero_()
dl.fused(*args, keep=keep, norm=norm)
torch.cuda.synchronize()
d = dbg.cpu().tolist()
names = ["row top (rec load)", "pass1 compute", "S1 wait", "send partial", "finish_row", "pass1 data wait", "masked zero-fill", "pass2"]
kept, rows = d[8], d[9]
print("kept rows (sum over CTAs)", kept, "rows", rows)
for i, n in enumerate(names):
    print(f"{n:22s} {d[i] / max(kept, 1):10.0f} cycles per kept row (avg over CTAs)")
