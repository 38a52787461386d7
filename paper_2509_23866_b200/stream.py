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

All arithmetic runs in the CUDA library; this module only sequences the ABI
calls and owns the buffers.
"""
from __future__ import annotations

import ctypes
from typing import Callable, List, Optional

import numpy as np
import torch

from . import dart
from .dart import DART_BF16, DART_F32, Shard, _check, _ptr


def chunk_layout(layout, max_rows: int) -> List[Shard]:
    """Greedy split into contiguous ranges of whole trajectories with at most
    `max_rows` token rows each (a single longer trajectory gets its own chunk)."""
    tso = np.asarray(layout.traj_step_off, dtype=np.int64)
    sto = np.asarray(layout.step_tok_off, dtype=np.int64)
    shards = []
    a = 0
    while a < layout.N_traj:
        b = a + 1
        while b < layout.N_traj and sto[tso[b + 1]] - sto[tso[a]] <= max_rows:
            b += 1
        s0, s1 = int(tso[a]), int(tso[b])
        shards.append(Shard(a, b, s0, s1, int(sto[s0]), int(sto[s1])))
        a = b
    return shards


class StreamedPass:
    def __init__(self, layout, V: int, cfg: dart.Config, device, max_rows: int, pool: int = 3,
                 logits_dtype=torch.bfloat16, grad_dtype=torch.bfloat16):
        self.L = dart.lib()
        dev = torch.device(device)
        self.device, self.layout, self.V, self.cfg = dev, layout, int(V), cfg
        self.logits_dtype, self.grad_dtype = logits_dtype, grad_dtype
        self.meta = dart.Meta.from_layout(layout, dev)
        self.chunks = chunk_layout(layout, max_rows)
        self.rows = max(c.T_loc for c in self.chunks)
        self.P = min(pool, len(self.chunks))
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
        self.S_pad = max(max(c.S_loc for c in self.chunks), 1)
        self.gathered = torch.zeros(n * self.S_pad, **f32)
        self.rank_step_off = torch.tensor([c.step_begin for c in self.chunks] + [self.chunks[-1].step_end],
                                          dtype=torch.int64, device=dev)
        self.stats_all = torch.zeros((n, len(dart.STATS_FIELDS)), dtype=torch.float64, device=dev)
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
        """target / log-prob inputs are global [T] device tensors.  fill(c, buf)
        must write chunk c's logits into buf[:T_c] (None: the pool slot already
        holds them).  consume(c, dlogits) gets a view of chunk c's gradient."""
        s = torch.cuda.current_stream(self.device).cuda_stream
        meta, cfg = ctypes.byref(self.meta.c()), ctypes.byref(self.cfg.c())
        beta = self.cfg.beta_kl > 0
        batches = []
        for i, c in enumerate(self.chunks):           # sweep 1: forward over every chunk
            buf = self.pool_logits[i % self.P]
            if fill is not None:
                fill(i, buf)
            sl = slice(c.tok_begin, c.tok_end)
            b = self._batch(c, buf, target[sl], logp_old[sl], logp_roll[sl], logp_ref[sl] if beta else None)
            batches.append(b)
            st = self.state[i]
            _check(self.L.dart_loss_fwd(ctypes.byref(b), meta, cfg, ctypes.byref(self._out(st)), _ptr(st["ws"]),
                                        st["ws_bytes"], ctypes.c_void_p(s)))
            self.launches += self.L.dart_last_launch_count()
            self.gathered[i * self.S_pad: i * self.S_pad + c.S_loc].copy_(st["step_H"][:c.S_loc])
        st0 = self.state[0]                            # select once (chunk 0's ws holds the group table)
        _check(self.L.dart_select_steps(_ptr(self.gathered), _ptr(self.rank_step_off), len(self.chunks),
                                        self.S_pad, meta, cfg, _ptr(self.group_ok), _ptr(self.keep),
                                        _ptr(self.tau), _ptr(self.norm), _ptr(st0["ws"]), st0["ws_bytes"],
                                        ctypes.c_void_p(s)))
        self.launches += self.L.dart_last_launch_count()
        gdt = DART_BF16 if self.grad_dtype == torch.bfloat16 else DART_F32
        for i, c in enumerate(self.chunks):           # sweep 2: gradient over every chunk
            if fill is not None and len(self.chunks) > self.P:
                fill(i, self.pool_logits[i % self.P])  # re-materialise an evicted chunk
            out = self.pool_dlogits[i % self.P]
            st = self.state[i]
            _check(self.L.dart_loss_bwd(ctypes.byref(batches[i]), meta, cfg, ctypes.byref(self._out(st)),
                                        _ptr(self.keep), _ptr(self.norm), _ptr(out), gdt, self.V,
                                        _ptr(self.stats_all[i]), _ptr(st["ws"]), st["ws_bytes"],
                                        ctypes.c_void_p(s)))
            self.launches += self.L.dart_last_launch_count()
            if consume is not None:
                consume(i, out[:c.T_loc])
        return self.stats_all

    def stats_dict(self):
        tot = self.stats_all.sum(dim=0).cpu().tolist()
        return dict(zip(dart.STATS_FIELDS, tot))

    def check_status(self):
        v = int(self.status.item())
        if v:
            names = [n for bit, n in dart.STATUS_BITS.items() if v & bit]
            raise dart.DartError(f"DART device status 0x{v:x}: {', '.join(names)}")
