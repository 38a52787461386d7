"""Stand-in for the N > 1 path on one GPU: shard a batch into W trajectory
ranges, run the three ABI calls per shard with the all-gather emulated by
concatenation; the assembled shards must pass compare() against the float64
oracle, and equal the unsharded pass bitwise (masks, counts, per-token
values, dlogits) -- the canonical reduction order makes the result
independent of the distribution -- with the loss to 1e-12."""
import numpy as np
import pytest
import torch

from paper_2509_23866_b200 import dart, synth
from paper_2509_23866_b200 import dist as D
from tests.gpu_helpers import Assembled, compare, run_gpu, snapshot

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,W", [("small_multi", 2), ("small_multi", 3), ("mid", 2), ("mid", 4),
                                    ("adaptive_small", 4)])
def test_sharded_equals_unsharded(name, W):
    if name == "adaptive_small":
        layout, _, _, _ = synth.config_layout("adaptive", seed=5)
        # keep the first 4 groups to bound the size
        nt = int(np.sum(layout.traj_group < 4))
        S = int(layout.traj_step_off[nt])
        layout = synth.Layout(G=4, traj_group=layout.traj_group[:nt], traj_reward=layout.traj_reward[:nt],
                              traj_step_off=layout.traj_step_off[:nt + 1], step_tok_off=layout.step_tok_off[:S + 1],
                              step_fork=layout.step_fork[:S])
        b = synth.make_batch("adaptive", seed=5, layout=layout, V=4096, dtype=torch.bfloat16)
    else:
        b = synth.make_batch(name, seed=2)
    cfg = dart.Config()
    ref = run_gpu(b, cfg)
    ref.check_status()
    shards = D.shard_layout(b.layout, W)
    dev = torch.device("cuda")
    gd = ref.grad_dtype
    dls = []
    for sh in shards:
        dl = dart.DartLoss(b.layout, sh, b.V, cfg, dev, logits_dtype=b.logits.dtype, grad_dtype=gd,
                           group=False, world_shards=shards)
        sl = slice(sh.tok_begin, sh.tok_end)
        dl.forward(b.logits[sl].to(dev).contiguous(), b.target[sl].to(dev).contiguous(),
                   b.logp_old[sl].to(dev).contiguous(), b.logp_rollout[sl].to(dev).contiguous(),
                   b.logp_ref[sl].to(dev).contiguous())
        dls.append(dl)
    S_pad = dls[0].S_pad
    gathered = torch.zeros(W * S_pad, dtype=torch.float32, device=dev)
    for r, (dl, sh) in enumerate(zip(dls, shards)):
        gathered[r * S_pad: r * S_pad + sh.S_loc] = dl.step_H[:sh.S_loc]
    loss = 0.0
    for dl, sh in zip(dls, shards):
        dl.set_gathered(gathered)
        dl.select()
        dl.backward()
    torch.cuda.synchronize()
    for dl, sh in zip(dls, shards):
        dl.check_status()
        sl = slice(sh.tok_begin, sh.tok_end)
        assert torch.equal(dl.keep[:b.layout.S], ref.keep[:b.layout.S])
        assert dl.norm_dict() == ref.norm_dict()
        for a, c in ((dl.lse, ref.lse[sl]), (dl.H, ref.H[sl]), (dl.ell, ref.ell[sl]), (dl.dell, ref.dell[sl])):
            assert torch.equal(a, c)
        assert torch.equal(dl.step_H[:sh.S_loc], ref.step_H[sh.step_begin:sh.step_end])
        assert torch.equal(dl.dlogits, ref.dlogits[sl])
        loss += dl.stats_dict()["loss"]
    L = ref.stats_dict()["loss"]
    assert abs(loss - L) <= 1e-12 * max(abs(L), 1e-30) + 1e-15
    rows = None
    if b.V > 4096:
        rows = sorted(np.random.default_rng(W).choice(b.layout.T, 16, replace=False).tolist())
    compare(Assembled([snapshot(dl, rows) for dl in dls], b.layout, grad_dtype=gd, stats_reduced=False),
            b, cfg, rows=rows)
