import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_23866_b200 import dart, synth
from oracle import dart_oracle as O
name = os.environ.get("CFG", "grid1x2x2x16@2048")
lb = synth.make_lmhead(name, int(os.environ.get("D", "64")), seed=1, exact=True)
b = lb.batch
dl = dart.DartLoss(b.layout, dart.whole_shard(b.layout), b.V, dart.Config(), "cuda", with_grad=False)
dl.forward_lmhead(lb.hidden.cuda(), lb.weight.cuda(), b.target.cuda(), b.logp_old.cuda(), b.logp_rollout.cuda(), b.logp_ref.cuda())
torch.cuda.synchronize()
print("status", int(dl.status.item()), flush=True)
ob = b.oracle_dict(logits=False)
ob["logits"] = O.lmhead_logits(lb.hidden.float().numpy(), lb.weight.float().numpy())
ref = O.loss_pass(ob, dart.Config().as_f32(), want_grad=False)
H = dl.H.cpu().numpy()
print("T", b.layout.T, "max H err", np.abs(H - ref["H"]).max(), "max lse err", np.abs(dl.lse.cpu().numpy() - ref["lse"]).max(), flush=True)
