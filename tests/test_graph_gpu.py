"""CUDA-graph capture of one whole pass (DartLoss.capture): replaying the graph
reproduces the eager pass bitwise (dlogits, mask, normaliser, statistics)."""
import pytest
import torch

from paper_2509_23866_b200 import dart, synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["mid", "small_multi"])
def test_graph_replay_equals_eager(name):
    b = synth.make_batch(name, seed=2, device="cuda")
    cfg = dart.Config()
    gd = torch.float32 if b.logits.dtype == torch.float32 else torch.bfloat16
    dl = dart.DartLoss(b.layout, dart.whole_shard(b.layout), b.V, cfg, "cuda", logits_dtype=b.logits.dtype,
                       grad_dtype=gd)
    inp = (b.logits, b.target, b.logp_old, b.logp_rollout, b.logp_ref)
    dl.run(*inp)
    torch.cuda.synchronize()
    ref = (dl.dlogits.clone(), dl.keep.clone(), dl.norm.clone(), dl.stats.clone(), dl.lse.clone())
    g = dl.capture(*inp)
    dl.dlogits_store.fill_(float("nan"))
    dl.lse.fill_(float("nan"))
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    dl.check_status()
    assert torch.equal(dl.dlogits, ref[0])
    assert torch.equal(dl.keep, ref[1]) and torch.equal(dl.norm, ref[2])
    assert torch.equal(dl.lse, ref[4])
    assert torch.equal(dl.stats, ref[3])
