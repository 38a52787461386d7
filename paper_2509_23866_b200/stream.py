"""Chunk-streamed DART pass for batches whose logits do not fit in HBM
(the long-horizon config is 249 GB of bf16 logits at one
GPU, the scale sweep up to 5.1 TB).

The token-mean normaliser needs every step's keep bit before any gradient,
so the schedule is

    fwd sweep over all chunks  ->  select once over the global step entropies
                               ->  bwd sweep over all chunks

Chunks are contiguous ranges of whole trajectories (they are exactly the
"virtual ranks" of the sharded path: the per-chunk step entropies are laid
out like an all-gather and `dart_select_steps` runs once).  Logits and
dlogits live in a pool of P device buffers: chunk c uses pool slot c mod P in
both sweeps.  The caller's `fill(c, buf)` writes chunk c's logits into its
slot (e.g. from the LM head or a host copy); for throughput measurement the
bench fills each slot once and re-uses it, which keeps both sweeps reading
identical bytes.  `consume(c, dlogits)` receives each chunk's gradient.

Across ranks (`group`): rank r streams the chunks of its own shard (a
contiguous, token-balanced range of whole trajectories, `dist.shard_layout`).
Every rank's chunks are the virtual ranks of ONE global selection: rank r
owns virtual ranks [r*C_max, (r+1)*C_max) (C_max = the largest per-rank chunk
count; missing ones are empty), so C1 is a single all-gather of each rank's
[C_max, S_pad] step-entropy block, `dart_select_steps` then yields the same
keep bits and normaliser on every rank, and C2 all-reduces the statistics.

All arithmetic runs in the CUDA library; this module only sequences the ABI
calls and owns the buffers.
"""
from __future__ import annotations

import ctypes
import dataclasses
from typing import Callable, List, Optional

import numpy as np
import torch

from . import dart
from .dart import DART_BF16, DART_F32, Shard, _check, _ptr


def chunk_layout(layout, max_rows: int, traj_begin: int = 0, traj_end: Optional[int] = None) -> List[Shard]:
    """Greedy split of trajectories [traj_begin, traj_end) into contiguous
    ranges of whole trajectories with at most `max_rows` token rows each (a
    single longer trajectory gets its own chunk)."""
    tso = np.asarray(layout.traj_step_off, dtype=np.int64)
    sto = np.asarray(layout.step_tok_off, dtype=np.int64)
    end = layout.N_traj if traj_end is None else int(traj_end)
    shards = []
    a = int(traj_begin)
    while a < end:
        b = a + 1
        while b < end and sto[tso[b + 1]] - sto[tso[a]] <= max_rows:
            b += 1
        s0, s1 = int(tso[a]), int(tso[b])
        shards.append(Shard(a, b, s0, s1, int(sto[s0]), int(sto[s1])))
        a = b
    return shards


def virtual_ranks(layout, world_shards: List[Shard], max_rows: int):
    """Chunks of every rank and the global virtual-rank table: returns
    (chunks per rank, C_max, S_pad, rank_step_off [world*C_max + 1]); rank r's
    chunk j is virtual rank r*C_max + j, missing ones are empty (no steps)."""
    per = [chunk_layout(layout, max_rows, sh.traj_begin, sh.traj_end) or [sh] for sh in world_shards]
    # (a rank without trajectories keeps one empty chunk: its forward call
    # still builds the global group tables the selection reads)
    c_max = max(1, max(len(c) for c in per))
    s_pad = max(1, max((c.S_loc for cs in per for c in cs), default=1))
    off = []
    for sh, cs in zip(world_shards, per):
        off.extend([c.step_begin for c in cs] + [sh.step_end] * (c_max - len(cs)))
    off.append(int(layout.S))
    return per, c_max, s_pad, np.asarray(off, dtype=np.int64)


class StreamedPass:
    def __init__(self, layout, V: int, cfg: dart.Config, device, max_rows: int, pool: int = 3,
                 logits_dtype=torch.bfloat16, grad_dtype=torch.bfloat16, group=None,
                 world_shards: Optional[List[Shard]] = None):
        if cfg.kl_mode == dart.KL_EXACT and cfg.beta_kl > 0:
            # the pool holds only the policy's logits; the exact KL would also need the
            # reference policy's rows streamed per chunk
            raise dart.DartError("the streamed pass supports the k3 KL only (kl_mode=KL_K3 or beta_kl=0)")
        self.L = dart.lib()
        dev = torch.device(device)
        # every chunk's dart_loss_bwd adds its loss / statistics into self.stats (in chunk order)
        self.device, self.layout, self.V = dev, layout, int(V)
        self.cfg = dataclasses.replace(cfg, stats_accumulate=1)
        self.logits_dtype, self.grad_dtype = logits_dtype, grad_dtype
        self.meta = dart.Meta.from_layout(layout, dev)
        self.group = group
        if group is not None:
            import torch.distributed as tdist
            from . import dist as D
            self.world, self.rank = tdist.get_world_size(group), tdist.get_rank(group)
            world_shards = world_shards or D.shard_layout(layout, self.world)
        else:
            self.world, self.rank = 1, 0
            world_shards = world_shards or [dart.whole_shard(layout)]
        if len(world_shards) != self.world:
            raise dart.DartError("world_shards must hold one shard per rank")
        self.shard = world_shards[self.rank]
        per, self.C_max, self.S_pad, rso = virtual_ranks(layout, world_shards, max_rows)
        self.chunks = per[self.rank]
        self.rows = max([c.T_loc for c in self.chunks] + [1])
        self.P = max(1, min(pool, len(self.chunks)))
        self.pool_logits = [torch.empty((self.rows, self.V), dtype=logits_dtype, device=dev) for _ in range(self.P)]
        self.pool_dlogits = [torch.empty((self.rows, self.V), dtype=grad_dtype, device=dev) for _ in range(self.P)]
        f32 = dict(dtype=torch.float32, device=dev)
        # global outputs shared by all chunks
        self.adv = torch.empty(max(layout.N_traj, 1), **f32)
        self.group_ok = torch.empty(max(layout.G, 1), dtype=torch.uint8, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.keep = torch.empty(max(layout.S, 1), dtype=torch.uint8, device=dev)
        self.tau = torch.empty(max(layout.G, 1), **f32)
        self.norm = torch.empty(5, dtype=torch.int64, device=dev)
        n = len(self.chunks)
        self.n_virtual = self.world * self.C_max
        self.local_H = torch.zeros(self.C_max * self.S_pad, **f32)       # this rank's block of C1
        self.gathered = torch.zeros(self.n_virtual * self.S_pad, **f32)
        self.rank_step_off = torch.as_tensor(rso, dtype=torch.int64).to(dev)
        self.stats = torch.zeros(len(dart.STATS_FIELDS), dtype=torch.float64, device=dev)
        # per-chunk state: forward outputs + workspace (tens of bytes per token)
        self.state = []
        for c in self.chunks:
            st = dict(lse=torch.empty(c.T_loc, **f32), logp=torch.empty(c.T_loc, **f32),
                      H=torch.empty(c.T_loc, **f32), ell=torch.empty(c.T_loc, **f32),
                      dell=torch.empty(c.T_loc, **f32), step_H=torch.empty(max(c.S_loc, 1), **f32),
                      step_ell=torch.empty(max(c.S_loc, 1), dtype=torch.float64, device=dev))
            b = self._batch(c, None, None, None, None, None)
            st["ws_bytes"] = int(self.L.dart_workspace_size(ctypes.byref(b), ctypes.byref(self.meta.c()),
                                                            ctypes.byref(cfg.c())))
            st["ws"] = torch.empty(st["ws_bytes"], dtype=torch.uint8, device=dev)
            self.state.append(st)
        self.launches = 0

    def _batch(self, c: Shard, logits, target, lo, lr, lref):
        dt = DART_BF16 if self.logits_dtype == torch.bfloat16 else DART_F32
        return dart.dart_batch(_ptr(logits), dt, c.T_loc, self.V, self.V, c.tok_begin, c.step_begin, c.S_loc,
                               _ptr(target), _ptr(lo), _ptr(lr), _ptr(lref))

    def _out(self, st):
        return dart.dart_fwd_out(_ptr(st["lse"]), _ptr(st["logp"]), _ptr(st["H"]), _ptr(st["ell"]),
                                 _ptr(st["dell"]), _ptr(st["step_H"]), _ptr(st["step_ell"]), _ptr(self.adv),
                                 _ptr(self.group_ok), _ptr(self.status))

    def run(self, target, logp_old, logp_roll, logp_ref, fill: Optional[Callable] = None,
            consume: Optional[Callable] = None):
        """target / log-prob inputs are this rank's [T_loc] device tensors
        (the whole batch when single-process; row 0 = the shard's first
        token).  fill(c, buf) must write local chunk c's logits into buf[:T_c]
        (None: the pool slot already holds them).  consume(c, dlogits) gets a
        view of chunk c's gradient.  Returns the (all-reduced) statistics."""
        s = torch.cuda.current_stream(self.device).cuda_stream
        meta, cfg = ctypes.byref(self.meta.c()), ctypes.byref(self.cfg.c())
        beta = self.cfg.beta_kl > 0
        base = self.shard.tok_begin
        batches = []
        for i, c in enumerate(self.chunks):           # sweep 1: forward over every chunk
            buf = self.pool_logits[i % self.P]
            if fill is not None:
                fill(i, buf)
            sl = slice(c.tok_begin - base, c.tok_end - base)
            b = self._batch(c, buf, target[sl], logp_old[sl], logp_roll[sl], logp_ref[sl] if beta else None)
            batches.append(b)
            st = self.state[i]
            _check(self.L.dart_loss_fwd(ctypes.byref(b), meta, cfg, ctypes.byref(self._out(st)), _ptr(st["ws"]),
                                        st["ws_bytes"], ctypes.c_void_p(s)))
            self.launches += self.L.dart_last_launch_count()
            self.local_H[i * self.S_pad: i * self.S_pad + c.S_loc].copy_(st["step_H"][:c.S_loc])
        if self.world > 1:                             # C1: one all-gather of every rank's block
            from . import dist as D
            D.all_gather_into(self.gathered, self.local_H, group=self.group)
        else:
            self.gathered.copy_(self.local_H)
        st0 = self.state[0]                            # select once (chunk 0's ws holds the group table)
        _check(self.L.dart_select_steps(_ptr(self.gathered), _ptr(self.rank_step_off), self.n_virtual,
                                        self.S_pad, meta, cfg, _ptr(self.group_ok), _ptr(self.keep),
                                        _ptr(self.tau), _ptr(self.norm), _ptr(st0["ws"]), st0["ws_bytes"],
                                        ctypes.c_void_p(s)))
        self.launches += self.L.dart_last_launch_count()
        gdt = DART_BF16 if self.grad_dtype == torch.bfloat16 else DART_F32
        self.stats.zero_()
        for i, c in enumerate(self.chunks):           # sweep 2: gradient over every chunk
            if fill is not None and len(self.chunks) > self.P:
                fill(i, self.pool_logits[i % self.P])  # re-materialise an evicted chunk
            out = self.pool_dlogits[i % self.P]
            st = self.state[i]
            _check(self.L.dart_loss_bwd(ctypes.byref(batches[i]), meta, cfg, ctypes.byref(self._out(st)),
                                        _ptr(self.keep), _ptr(self.norm), _ptr(out), gdt, self.V,
                                        _ptr(self.stats), _ptr(st["ws"]), st["ws_bytes"],
                                        ctypes.c_void_p(s)))
            self.launches += self.L.dart_last_launch_count()
            if consume is not None:
                consume(i, out[:c.T_loc])
        if self.world > 1:                             # C2: statistics all-reduce
            from . import dist as D
            D.all_reduce(self.stats, group=self.group)
        return self.stats

    def stats_dict(self):
        return dict(zip(dart.STATS_FIELDS, self.stats.cpu().tolist()))

    def check_status(self):
        v = int(self.status.item())
        if v:
            names = [n for bit, n in dart.STATUS_BITS.items() if v & bit]
            raise dart.DartError(f"DART device status 0x{v:x}: {', '.join(names)}")
