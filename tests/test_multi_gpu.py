"""The N > 1 code path -- DartLoss.run with a process group doing C1 (the
step-entropy all-gather) and C2 (the statistics all-reduce) -- with the
ranks' results assembled and compared with the float64 ORACLE on the whole
batch (App. A.4: data-parallel trainer).

* nccl, W = 2 / 4 / 8: one rank per GPU over NVLink, as `bench.py --gpus W`
  runs it; skipped when fewer than W GPUs are visible.
* gloo, W = 2 / 3: the same code with the ranks sharing cuda:0 and the
  collectives staged through host memory (runs on a 1-GPU box).

Every rank must hold bitwise-identical replicated values (group_ok, A, keep,
tau, normaliser, all-reduced statistics); the assembled per-token values,
step entropies, mask, loss and every dlogits row must pass compare() against
the oracle.  The adaptive recipe (ragged groups of 2-8 rollouts, caps 2-8
steps, 4-40 tokens per step) makes task groups straddle ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2509_23866_b200 import dart, synth
from tests.gpu_helpers import Assembled, compare, snapshot

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg(name):
    if name.startswith("fuzz/"):       # a randomised case of tests/test_fuzz_gpu.py
        from tests.test_fuzz_gpu import _make
        return _make(int(name[5:]))[2]
    return dart.Config(is_cap=2.0) if name.startswith("tiny") else dart.Config()


def _batch(name, seed):
    if name.startswith("fuzz/"):
        from tests.test_fuzz_gpu import _make
        return _make(int(name[5:]))[0]
    _, V, dt, _ = synth.config_layout(name, seed)
    per = 16 // (2 if dt == torch.bfloat16 else 4)
    return synth.make_batch(name, seed=seed, pad_ld=-(-V // per) * per)


def _rows(name, seed, sample, T, starts):
    if not sample:
        return None
    rng = np.random.default_rng(seed)
    return sorted(set(rng.choice(T, sample, replace=False).tolist()) | set(starts))


def _worker(rank, world, backend, port, name, seed, sample, q):
    import torch.distributed as dist
    from paper_2509_23866_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", rank if backend == "nccl" else 0)
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b = _batch(name, seed)                          # CPU generator: identical bits on every rank
        shards = D.shard_layout(b.layout, world)
        me = shards[rank]
        ld = b.logits_store.stride(0)                   # 16-byte aligned rows (odd V is padded)
        dl = dart.DartLoss(b.layout, me, b.V, _cfg(name), dev, logits_dtype=b.logits.dtype,
                           grad_dtype=torch.bfloat16, group=dist.group.WORLD, world_shards=shards, ld=ld)
        sl = slice(me.tok_begin, me.tok_end)
        dl.run(b.logits_store[sl].to(dev)[:, :b.V],
               *(x[sl].to(dev).contiguous() for x in (b.target, b.logp_old, b.logp_rollout, b.logp_ref)))
        torch.cuda.synchronize()
        rows = _rows(name, seed, sample, b.layout.T, [s.tok_begin for s in shards if s.T_loc])
        q.put((rank, snapshot(dl, rows)))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(backend, world, name, seed, sample=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, backend, port, name, seed, sample, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=900) for _ in ps]
    for p in ps:
        p.join(timeout=120)
    for r, s in res:
        assert isinstance(s, dict), f"rank {r}: {s}"
    return [s for _, s in res]


CASES = [("adaptive_mini", 0, None), ("adaptive_mini", 1, None), ("mid", 3, 24)]


def _check(parts, name, seed, sample):
    b = _batch(name, seed)
    cfg = _cfg(name)
    view = Assembled(parts, b.layout)
    owners = {}
    for r, p in enumerate(parts):
        for i in range(*p["traj"]):
            owners.setdefault(int(b.layout.traj_group[i]), set()).add(r)
    if name != "mid" and not name.startswith("fuzz/"):   # adaptive mix / tiny over 5 ranks: groups straddle ranks
        assert any(len(rs) > 1 for rs in owners.values())
    rows = _rows(name, seed, sample, b.layout.T, [p["tok"][0] for p in parts if p["tok"][1] > p["tok"][0]])
    compare(view, b, cfg, rows=rows)


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name,seed,sample", CASES)
def test_nccl_ranks_vs_oracle(world, name, seed, sample):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (one NCCL rank per GPU), found {torch.cuda.device_count()}")
    _check(_run("nccl", world, name, seed, sample), name, seed, sample)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name,seed,sample", CASES[:1] + CASES[2:])
def test_gloo_ranks_one_gpu_vs_oracle(world, name, seed, sample):
    _check(_run("gloo", world, name, seed, sample), name, seed, sample)


def test_gloo_more_ranks_than_trajectories():
    """5 ranks for the tiny config's 4 trajectories: one rank owns nothing,
    still takes part in both collectives and holds the global mask."""
    from paper_2509_23866_b200 import dist as D
    assert any(s.T_loc == 0 for s in D.shard_layout(synth.make_batch("tiny", seed=1).layout, 5))
    _check(_run("gloo", 5, "tiny", 1), "tiny", 1, None)


@pytest.mark.parametrize("seed,world", [(11, 2), (23, 3), (42, 4)])
def test_gloo_ranks_one_gpu_fuzz_vs_oracle(seed, world):
    """Randomised batches of tests/test_fuzz_gpu.py (ragged groups, odd / padded
    vocabularies, -inf entries, random configurations) over real gloo process
    groups sharing one GPU: the collectives' padding and empty shards on
    random layouts, every rank checked against the oracle."""
    name = f"fuzz/{seed}"
    _check(_run("gloo", world, name, seed), name, seed, None)
