import sys; sys.path.insert(0,'.')
import numpy as np, torch
from oracle import dart_oracle as O
from paper_2509_23866_b200 import dart, lmhead, synth
from tests.test_lmhead_update_gpu import old_pass, run_update
lb = synth.make_lmhead("grid3x4x3x24@3000", 256, seed=21)
cfg = dart.Config(entropy_q=0.3, eps_low=0.95, eps_high=0.95)
old = old_pass(lb, cfg)
up, dh, dW = run_update(lb, cfg, old.keep, old.norm, 200)
cfgf = cfg.as_f32()
L = lb.batch.layout
h, W = lb.hidden.float().numpy(), lb.weight.float().numpy()
ob = lb.batch.oracle_dict(logits=False); ob["logits"] = O.lmhead_logits(h, W)
keep = old.keep.cpu().numpy()[:L.S]
ref = O.loss_pass(ob, cfgf, keep_override=keep)
dz = np.stack([ref["dz"][t] for t in range(L.T)])
dh_ref, dW_ref = O.lmhead_grads(dz, h, W)
dhg = dh.cpu().numpy()
print("keep", keep[:6], "chunks", [(c.tok_begin, c.tok_end) for c in up.chunks][:4])
for t in [0, 5, 23, 24, 25, 47, 48, 100, 143, 144]:
    print(t, "gpu", dhg[t, :3], "ref", dh_ref[t, :3], "dell", ref["dell"][t], up.dell[t].item(), "c", ref["c_tok"][t], "lse", ref["lse"][t], up.lse[t].item(), old.lse[t].item())
