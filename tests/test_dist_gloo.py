"""Host side of the N > 1 path on CPU with gloo, world size 2: trajectory
sharding, the padded step-entropy all-gather layout that dart_select_steps
takes (include/dart_loss.h), and the fp64 statistics all-reduce."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_23866_b200 import dist as D
from paper_2509_23866_b200 import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        layout, _, _, _ = synth.config_layout(name, seed=3)
        shards = D.shard_layout(layout, world)
        me = shards[rank]
        S_pad = D.s_pad(shards)
        # stand-in for the step entropies: the global step index as float
        local = torch.arange(me.step_begin, me.step_end, dtype=torch.float32)
        gathered = D.gather_padded(local, S_pad)
        # the layout contract: rank r's steps at [r*S_pad, r*S_pad + S_loc_r)
        g = gathered.numpy()
        for r, sh in enumerate(shards):
            assert np.array_equal(g[r * S_pad: r * S_pad + sh.S_loc], np.arange(sh.step_begin, sh.step_end))
        stats = torch.tensor([float(me.T_loc), float(me.S_loc), 0.5 * (rank + 1)], dtype=torch.float64)
        D.reduce_stats(stats)
        assert stats[0].item() == layout.T and stats[1].item() == layout.S
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["small_multi", "adaptive"])
def test_gloo_world2_gather_layout(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("name", ["single", "adaptive", "small_multi", "long"])
def test_shards_cover_whole_trajectories_balanced(name, world):
    layout, _, _, _ = synth.config_layout(name, seed=0)
    shards = D.shard_layout(layout, world)
    assert shards[0].traj_begin == 0 and shards[-1].traj_end == layout.N_traj
    for a, b in zip(shards, shards[1:]):
        assert a.traj_end == b.traj_begin and a.step_end == b.step_begin and a.tok_end == b.tok_begin
    for s in shards:
        assert s.step_begin == layout.traj_step_off[s.traj_begin]
        assert s.tok_begin == layout.step_tok_off[s.step_begin]
    # token balance within one (largest) trajectory of the ideal share
    tso, sto = layout.traj_step_off, layout.step_tok_off
    max_traj = int(np.max(sto[tso[1:]] - sto[tso[:-1]]))
    for s in shards:
        if layout.N_traj >= world:
            assert abs(s.T_loc - layout.T / world) <= max_traj


def test_chunk_layout_whole_trajectories():
    from paper_2509_23866_b200.stream import chunk_layout
    layout, _, _, _ = synth.config_layout("long", seed=0)
    ch = chunk_layout(layout, 32768)
    assert ch[0].tok_begin == 0 and ch[-1].tok_end == layout.T
    for a, c in zip(ch, ch[1:]):
        assert a.traj_end == c.traj_begin and a.tok_end == c.tok_begin
    assert max(c.T_loc for c in ch) <= 32768
