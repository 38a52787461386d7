"""Chunk-streamed pass (batches larger than HBM): forward over all
chunks -> one selection -> backward over all chunks, with a pool of P logits
buffers refilled per chunk.  Must reproduce the resident pass bitwise (mask,
counts, dlogits) and the loss to 1e-12."""
import numpy as np
import pytest
import torch

from paper_2509_23866_b200 import dart, synth
from paper_2509_23866_b200.stream import StreamedPass, chunk_layout
from tests.gpu_helpers import run_gpu

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("max_rows,pool", [(300, 2), (700, 3), (100000, 3)])
def test_streamed_equals_resident(max_rows, pool):
    b = synth.make_batch("mid", seed=4)
    cfg = dart.Config()
    ref = run_gpu(b, cfg)
    dev = torch.device("cuda")
    logits = b.logits.to(dev)
    sp = StreamedPass(b.layout, b.V, cfg, dev, max_rows=max_rows, pool=pool)
    assert len(sp.chunks) >= 1
    got = torch.empty_like(ref.dlogits)

    def fill(i, buf):
        c = sp.chunks[i]
        buf[:c.T_loc].copy_(logits[c.tok_begin:c.tok_end])

    def consume(i, dz):
        c = sp.chunks[i]
        got[c.tok_begin:c.tok_end].copy_(dz)

    sp.run(b.target.to(dev), b.logp_old.to(dev), b.logp_rollout.to(dev), b.logp_ref.to(dev), fill=fill,
           consume=consume)
    torch.cuda.synchronize()
    sp.check_status()
    assert torch.equal(sp.keep[:b.layout.S], ref.keep[:b.layout.S])
    assert torch.equal(sp.norm, ref.norm)
    assert torch.equal(got, ref.dlogits)
    L = ref.stats_dict()["loss"]
    assert abs(sp.stats_dict()["loss"] - L) <= 1e-12 * abs(L) + 1e-15
    assert sp.stats_dict()["n_kept_tok"] == ref.stats_dict()["n_kept_tok"]
