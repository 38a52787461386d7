"""Small driver for compute-sanitizer: one pass of a few configs through the C ABI."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2509_23866_b200 import dart, synth
from tests.gpu_helpers import run_gpu

which = sys.argv[1:] or ["tiny", "small_multi", "odd"]
for name in which:
    if name == "odd":
        layout, _, _, _ = synth.config_layout("small_multi", seed=1)
        b = synth.make_batch("small_multi", seed=1, layout=layout, V=1001, dtype=torch.bfloat16, pad_ld=1008)
    elif name == "midsplit":   # V = 152064, few rows -> split-row mode + bulk copies of full chunks
        layout, _, _, _ = synth.config_layout("grid1x2x2x16@152064", seed=0)
        b = synth.make_batch("x", seed=0, layout=layout, V=152064, dtype=torch.bfloat16)
    elif name == "lmhead":   # NEXT #3: tcgen05 / TMA / TMEM kernel + combine, ragged rows and vocabulary
        lb = synth.make_lmhead("grid2x4x3x20@3000", 256, seed=3, exact=True)
        bb = lb.batch
        dl = dart.DartLoss(bb.layout, dart.whole_shard(bb.layout), bb.V, dart.Config(), "cuda", with_grad=False)
        dl.forward_lmhead(lb.hidden.cuda(), lb.weight.cuda(), bb.target.cuda(), bb.logp_old.cuda(),
                          bb.logp_rollout.cuda(), bb.logp_ref.cuda())
        dl.select()
        dl.backward()
        torch.cuda.synchronize()
        dl.check_status()
        print(name, "ok", dl.stats_dict()["loss"])
        continue
    elif name == "lmupdate":   # NEXT #3 update pass: forward + dz from the z-GEMM epilogue (kept rows)
        from paper_2509_23866_b200 import lmhead
        lb = synth.make_lmhead("grid2x4x3x20@3000", 256, seed=3)
        bb = lb.batch
        old = dart.DartLoss(bb.layout, dart.whole_shard(bb.layout), bb.V, dart.Config(), "cuda", with_grad=False)
        args = (bb.target.cuda(), bb.logp_old.cuda(), bb.logp_rollout.cuda(), bb.logp_ref.cuda())
        old.forward_lmhead(lb.hidden.cuda(), lb.weight.cuda(), *args)
        old.select()
        up = lmhead.LmHeadUpdate(bb.layout, bb.V, 256, dart.Config(), "cuda", chunk_rows=150)
        dh, dW = up.run(lb.hidden.cuda(), lb.weight.cuda(), *args, old.keep, old.norm)
        torch.cuda.synchronize()
        up.check_status()
        print(name, "ok", up.stats_dict()["loss"], float(dh.abs().sum()), float(dW.abs().sum()))
        continue
    elif name == "fused":   # NEXT #1: the fused update kernel
        layout, _, _, _ = synth.config_layout("grid2x2x3x24@30000", seed=0)
        b = synth.make_batch("x", seed=0, layout=layout, V=30000, dtype=torch.bfloat16)
        old = run_gpu(b, dart.Config())
        dl = dart.DartLoss(b.layout, dart.whole_shard(b.layout), b.V, dart.Config(), "cuda")
        dl.fused(b.logits.cuda(), b.target.cuda(), b.logp_old.cuda(), b.logp_rollout.cuda(), b.logp_ref.cuda(),
                 keep=old.keep, norm=old.norm)
        torch.cuda.synchronize()
        dl.check_status()
        print(name, "ok", dl.stats_dict()["loss"])
        continue
    elif name == "klexact":  # NEXT #4
        b = synth.make_batch("small_multi", seed=0, with_ref=True)
        dl = dart.DartLoss(b.layout, dart.whole_shard(b.layout), b.V, dart.Config(kl_mode=dart.KL_EXACT), "cuda",
                           logits_dtype=b.logits.dtype, grad_dtype=torch.float32 if b.logits.dtype == torch.float32 else torch.bfloat16)
        dl.run(b.logits.cuda(), b.target.cuda(), b.logp_old.cuda(), b.logp_rollout.cuda(), b.logp_ref.cuda(),
               b.ref_logits.cuda())
        torch.cuda.synchronize()
        dl.check_status()
        print(name, "ok", dl.stats_dict()["loss"])
        continue
    else:
        b = synth.make_batch(name, seed=0)
    dl = run_gpu(b, dart.Config(is_cap=2.0 if name.startswith("tiny") else 1.0))
    dl.check_status()
    print(name, "ok", dl.stats_dict()["loss"])
