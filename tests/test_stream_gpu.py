"""Chunk-streamed pass (batches larger than HBM): forward over all
chunks -> one selection -> backward over all chunks, with a pool of P logits
buffers refilled per chunk.  The streamed results (assembled over chunks and
ranks) must pass compare() against the float64 oracle, and reproduce the
resident pass bitwise (mask, counts, dlogits) and its loss to 1e-12."""
import numpy as np
import pytest
import torch

from paper_2509_23866_b200 import dart, synth
from paper_2509_23866_b200.stream import StreamedPass, chunk_layout
from tests.gpu_helpers import Assembled, compare, run_gpu, stream_snapshot


def _sample(b, seed, n=16):
    rng = np.random.default_rng(seed)
    return sorted(rng.choice(b.layout.T, n, replace=False).tolist())

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
    rows = _sample(b, max_rows)
    compare(Assembled([stream_snapshot(sp, got, rows)], b.layout), b, cfg, rows=rows)
    assert torch.equal(sp.keep[:b.layout.S], ref.keep[:b.layout.S])
    assert torch.equal(sp.norm, ref.norm)
    assert torch.equal(got, ref.dlogits)
    L = ref.stats_dict()["loss"]
    assert abs(sp.stats_dict()["loss"] - L) <= 1e-12 * abs(L) + 1e-15
    assert sp.stats_dict()["n_kept_tok"] == ref.stats_dict()["n_kept_tok"]


def _mr_worker(rank, world, port, max_rows, q, name="mid", seed=4):
    import os
    import torch.distributed as dist
    from paper_2509_23866_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        b = synth.make_batch(name, seed=seed)
        shards = D.shard_layout(b.layout, world)
        me = shards[rank]
        gd = torch.float32 if b.logits.dtype == torch.float32 else torch.bfloat16
        cfg = dart.Config(is_cap=2.0) if name == "tiny" else dart.Config()
        sp = StreamedPass(b.layout, b.V, cfg, dev, max_rows=max_rows, pool=2, group=dist.group.WORLD,
                          world_shards=shards, logits_dtype=b.logits.dtype, grad_dtype=gd)
        logits = b.logits.to(dev)
        got = torch.empty((me.T_loc, b.V), dtype=gd, device=dev)

        def fill(i, buf):
            c = sp.chunks[i]
            buf[:c.T_loc].copy_(logits[c.tok_begin:c.tok_end])

        def consume(i, dz):
            c = sp.chunks[i]
            got[c.tok_begin - me.tok_begin:c.tok_end - me.tok_begin].copy_(dz)

        sl = slice(me.tok_begin, me.tok_end)
        sp.run(*(x[sl].to(dev).contiguous() for x in (b.target, b.logp_old, b.logp_rollout, b.logp_ref)),
               fill=fill, consume=consume)
        torch.cuda.synchronize()
        sp.check_status()
        q.put((rank, got.view(torch.int16 if gd == torch.bfloat16 else torch.int32).cpu().numpy(),
               sp.keep.cpu().numpy(), sp.norm.cpu().numpy(),
               sp.stats_dict(), me.tok_begin, me.tok_end, len(sp.chunks),
               stream_snapshot(sp, got, _sample(b, 1) if b.V > 4096 else None)))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), None, None, None, 0, 0, 0, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("max_rows", [300, 100000])
def test_streamed_two_ranks_equal_resident(max_rows):
    """The multi-rank streamed pass (each rank streams its own shard's chunks,
    one all-gather of every rank's per-chunk step entropies, one selection,
    statistics all-reduce) with 2 ranks sharing one GPU through gloo: each
    rank's dlogits bitwise equal to the resident unsharded pass."""
    import socket
    import torch.multiprocessing as mp
    b = synth.make_batch("mid", seed=4)
    ref = run_gpu(b, dart.Config())
    ref_dz = ref.dlogits.view(torch.int16).cpu().numpy()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_mr_worker, args=(r, 2, port, max_rows, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    L = ref.stats_dict()["loss"]
    for rank, dz, keep, norm, st, t0, t1, nch, snap in res:
        assert keep is not None, dz
        assert np.array_equal(keep[:b.layout.S], ref.keep.cpu().numpy()[:b.layout.S])
        assert np.array_equal(norm, ref.norm.cpu().numpy())
        assert np.array_equal(dz, ref_dz[t0:t1])
        assert abs(st["loss"] - L) <= 1e-12 * abs(L) + 1e-15       # all-reduced on every rank
        assert st["n_kept_tok"] == ref.stats_dict()["n_kept_tok"]
    rows = _sample(b, 1)
    compare(Assembled([r[-1] for r in res], b.layout), b, dart.Config(), rows=rows)


def test_streamed_more_ranks_than_trajectories():
    """5 ranks for the tiny config's 4 trajectories: one rank owns nothing
    (one empty chunk; its forward call still builds the global group tables);
    every rank's gradient rows bitwise equal to the resident pass."""
    import socket
    import torch.multiprocessing as mp
    from paper_2509_23866_b200 import dist as D
    b = synth.make_batch("tiny", seed=1)
    ref = run_gpu(b, dart.Config(is_cap=2.0))
    assert any(s.T_loc == 0 for s in D.shard_layout(b.layout, 5))
    ref_dz = ref.dlogits.view(torch.int32).cpu().numpy()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_mr_worker, args=(r, 5, port, 40, q, "tiny", 1)) for r in range(5)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    L = ref.stats_dict()["loss"]
    for rank, dz, keep, norm, st, t0, t1, nch, snap in res:
        assert keep is not None, dz
        assert np.array_equal(keep[:b.layout.S], ref.keep.cpu().numpy()[:b.layout.S])
        assert np.array_equal(norm, ref.norm.cpu().numpy())
        assert np.array_equal(dz, ref_dz[t0:t1])
        assert abs(st["loss"] - L) <= 1e-12 * abs(L) + 1e-15
    compare(Assembled([r[-1] for r in res], b.layout, grad_dtype=torch.float32), b, dart.Config(is_cap=2.0))

