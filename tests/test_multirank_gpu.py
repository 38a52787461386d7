"""The real N > 1 code path -- DartLoss.run with a process group doing the
step-entropy all-gather and the statistics all-reduce -- with 2 ranks
sharing one GPU (gloo, collectives staged through host memory; the NCCL
path differs only in the backend).  Each rank's dlogits must equal the
unsharded pass bitwise and the all-reduced loss must match to 1e-12."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2509_23866_b200 import dart, synth
    from paper_2509_23866_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        b = synth.make_batch("mid", seed=3)
        shards = D.shard_layout(b.layout, world)
        me = shards[rank]
        cfg = dart.Config()
        dev = torch.device("cuda", 0)
        dl = dart.DartLoss(b.layout, me, b.V, cfg, dev, logits_dtype=b.logits.dtype, grad_dtype=torch.bfloat16,
                           group=dist.group.WORLD, world_shards=shards)
        sl = slice(me.tok_begin, me.tok_end)
        dl.run(b.logits[sl].to(dev).contiguous(), b.target[sl].to(dev).contiguous(),
               b.logp_old[sl].to(dev).contiguous(), b.logp_rollout[sl].to(dev).contiguous(),
               b.logp_ref[sl].to(dev).contiguous())
        torch.cuda.synchronize()
        dl.check_status()
        q.put((rank, dl.dlogits.view(torch.int16).cpu().numpy(), dl.keep.cpu().numpy(), dl.stats_dict(),
               me.tok_begin, me.tok_end))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), None, None, 0, 0))
    finally:
        dist.destroy_process_group()


def test_two_ranks_one_gpu_equal_unsharded():
    from paper_2509_23866_b200 import dart, synth
    from tests.gpu_helpers import run_gpu
    b = synth.make_batch("mid", seed=3)
    ref = run_gpu(b, dart.Config())
    ref_dz = ref.dlogits.view(torch.int16).cpu().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, dz, keep, st, t0, t1 in res:
        assert keep is not None, dz
        assert np.array_equal(keep, ref.keep.cpu().numpy())
        assert np.array_equal(dz, ref_dz[t0:t1])
        L = ref.stats_dict()["loss"]
        assert abs(st["loss"] - L) <= 1e-12 * abs(L) + 1e-15     # all-reduced on every rank
        assert st["n_kept_tok"] == ref.stats_dict()["n_kept_tok"]
