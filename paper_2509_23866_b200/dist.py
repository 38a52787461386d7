"""Data-parallel plumbing: trajectory sharding and the two collectives.

Trajectories shard across ranks as contiguous, token-balanced ranges of whole
trajectories (a trajectory's steps never straddle ranks; a task group may).
Every rank holds the global metadata, so advantages and the normaliser need
no communication; the only exchanges are
  C1  all_gather of the fp32 step entropies (padded to S_pad per rank), and
  C2  all_reduce(SUM) of the fp64 loss / statistics partials.
"""
from __future__ import annotations

import numpy as np
import torch

from .dart import Shard


def shard_layout(layout, world: int):
    """Split the N_traj trajectories into `world` contiguous ranges with
    near-equal token counts (greedy on the cumulative token count)."""
    tso = np.asarray(layout.traj_step_off, dtype=np.int64)
    sto = np.asarray(layout.step_tok_off, dtype=np.int64)
    traj_tok_end = sto[tso[1:]]            # cumulative tokens at the end of each trajectory
    T = int(sto[-1])
    bounds = [0]
    for r in range(1, world):
        target = T * r / world
        i = int(np.searchsorted(traj_tok_end, target, side="left"))
        # choose the trajectory boundary closest to the target
        cand = [c for c in (i, i + 1) if bounds[-1] <= c <= layout.N_traj]
        best = min(cand, key=lambda c: abs((traj_tok_end[c - 1] if c > 0 else 0) - target))
        bounds.append(max(best, bounds[-1]))
    bounds.append(layout.N_traj)
    shards = []
    for r in range(world):
        a, b = bounds[r], bounds[r + 1]
        s0, s1 = int(tso[a]), int(tso[b])
        shards.append(Shard(a, b, s0, s1, int(sto[s0]), int(sto[s1])))
    return shards


def s_pad(shards):
    return max(max(s.S_loc for s in shards), 1)


def _gloo(group=None):
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


def all_gather_into(out: torch.Tensor, inp: torch.Tensor, group=None):
    """all_gather_into_tensor; with gloo (CPU test backend) CUDA tensors are
    staged through host memory."""
    import torch.distributed as dist
    if out.is_cuda and _gloo(group):
        o = out.cpu()
        dist.all_gather_into_tensor(o, inp.cpu(), group=group)
        out.copy_(o)
    else:
        dist.all_gather_into_tensor(out, inp, group=group)
    return out


def all_reduce(t: torch.Tensor, op=None, group=None):
    import torch.distributed as dist
    op = dist.ReduceOp.SUM if op is None else op
    if t.is_cuda and _gloo(group):
        c = t.cpu()
        dist.all_reduce(c, op=op, group=group)
        t.copy_(c)
    else:
        dist.all_reduce(t, op=op, group=group)
    return t


def gather_padded(local: torch.Tensor, S_pad: int, group=None) -> torch.Tensor:
    """C1: every rank contributes `local` (its S_loc step values) padded to
    S_pad; returns [world * S_pad] in rank order (the layout
    dart_select_steps takes, include/dart_loss.h)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    pad = torch.zeros(S_pad, dtype=local.dtype, device=local.device)
    pad[:local.numel()].copy_(local)
    out = torch.empty(world * S_pad, dtype=local.dtype, device=local.device)
    all_gather_into(out, pad, group=group)
    return out


def reduce_stats(stats: torch.Tensor, group=None) -> torch.Tensor:
    """C2: all-reduce(SUM) of the fp64 loss / statistics partials."""
    return all_reduce(stats, group=group)
