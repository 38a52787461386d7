"""Host side of the multi-rank chunk-streamed pass (stream.virtual_ranks) on
CPU: every rank's chunks tile its shard with whole trajectories, the virtual
rank table is the all-gather layout dart_select_steps takes, and with gloo at
world size 2 the gathered per-rank blocks unpack to global step order."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_23866_b200 import dist as D
from paper_2509_23866_b200 import synth
from paper_2509_23866_b200.stream import chunk_layout, virtual_ranks


def _unpack(gathered, rso, S_pad, S):
    """include/dart_loss.h layout: virtual rank v's steps at [v*S_pad, v*S_pad + n_v)."""
    out = np.full(S, np.nan)
    for v in range(len(rso) - 1):
        n = rso[v + 1] - rso[v]
        out[rso[v]:rso[v + 1]] = gathered[v * S_pad: v * S_pad + n]
    return out


@pytest.mark.parametrize("name,world,max_rows", [("small_multi", 2, 40), ("small_multi", 3, 15),
                                                 ("adaptive", 8, 32768), ("adaptive", 3, 2000),
                                                 ("single", 2, 4096), ("tiny", 4, 64),
                                                 ("tiny", 6, 64)])
def test_virtual_rank_table(name, world, max_rows):
    L, _, _, _ = synth.config_layout(name, seed=1)
    shards = D.shard_layout(L, world)
    per, c_max, s_pad, rso = virtual_ranks(L, shards, max_rows)
    assert len(per) == world and len(rso) == world * c_max + 1
    assert rso[0] == 0 and rso[-1] == L.S and np.all(np.diff(rso) >= 0)
    sto, tso = np.asarray(L.step_tok_off), np.asarray(L.traj_step_off)
    for r, (sh, cs) in enumerate(zip(shards, per)):
        assert 1 <= len(cs) <= c_max
        # chunks tile the shard: contiguous whole trajectories, in order
        assert cs[0].traj_begin == sh.traj_begin and cs[-1].traj_end == sh.traj_end
        for a, b in zip(cs, cs[1:]):
            assert a.traj_end == b.traj_begin
        for j, c in enumerate(cs):
            assert c.step_begin == tso[c.traj_begin] and c.step_end == tso[c.traj_end]
            assert c.tok_begin == sto[c.step_begin] and c.tok_end == sto[c.step_end]
            assert c.T_loc <= max_rows or c.traj_end - c.traj_begin == 1
            assert c.S_loc <= s_pad
            assert rso[r * c_max + j] == c.step_begin and rso[r * c_max + j + 1] - rso[r * c_max + j] == c.S_loc
        for j in range(len(cs), c_max):          # padding virtual ranks are empty
            assert rso[r * c_max + j] == sh.step_end == rso[r * c_max + j + 1]
    # a single rank reproduces the one-process chunking
    per1, c1, _, rso1 = virtual_ranks(L, [D.shard_layout(L, 1)[0]], max_rows)
    assert [(c.traj_begin, c.traj_end) for c in per1[0]] == \
        [(c.traj_begin, c.traj_end) for c in chunk_layout(L, max_rows)]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, max_rows, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L, _, _, _ = synth.config_layout(name, seed=2)
        shards = D.shard_layout(L, world)
        per, c_max, s_pad, rso = virtual_ranks(L, shards, max_rows)
        # stand-in for each chunk's step entropies: the global step index
        local = torch.zeros(c_max * s_pad, dtype=torch.float32)
        for j, c in enumerate(per[rank]):
            local[j * s_pad: j * s_pad + c.S_loc] = torch.arange(c.step_begin, c.step_end, dtype=torch.float32)
        out = torch.empty(world * c_max * s_pad, dtype=torch.float32)
        D.all_gather_into(out, local)
        H = _unpack(out.numpy(), rso, s_pad, L.S)
        assert np.array_equal(H, np.arange(L.S, dtype=np.float64))
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,max_rows", [("small_multi", 30), ("adaptive", 20000)])
def test_gloo_world2_streamed_gather(name, max_rows):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, name, max_rows, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=30)
    assert sorted(res) == [(0, "ok"), (1, "ok")], res
