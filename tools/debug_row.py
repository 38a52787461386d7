import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2509_23866_b200 import dart, synth
from tests.gpu_helpers import run_gpu
from oracle import dart_oracle as O
b = synth.make_batch("small_multi", seed=0)
cfg = dart.Config(norm_mode=2, entropy_q=0.3)
dl = run_gpu(b, cfg)
t = 1037
ob = b.oracle_dict()
ref = O.loss_pass(ob, cfg.as_f32(), keep_override=dl.keep.cpu().numpy(), rows=[t])
y = int(b.target[t])
np.set_printoptions(precision=17)
print("y", y, "z_y", float(b.logits[t, y]), "max", float(b.logits[t].max()), "argmax", int(b.logits[t].argmax()))
for k in ("lse", "logp", "H", "ell", "dell"):
    print(k, repr(float(getattr(dl, k)[t])), repr(ref[k][t]))
print("logp_old", float(b.logp_old[t]), "logp_ref", float(b.logp_ref[t]), "roll", float(b.logp_rollout[t]))
print("c_tok", ref["c_tok"][t], "inv_norm", dl.norm_dict())
dz = dl.dlogits[t].cpu().numpy()
print("dz_y gpu", dz[y], "ref", ref["dz"][t][y])
print("dz others gpu/ref ratio", (dz[:5] / ref["dz"][t][:5]))
