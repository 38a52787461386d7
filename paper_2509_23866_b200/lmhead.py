"""LM-head-fused update pass (training half).

The forward half is `DartLoss.forward_lmhead` (dart_lmhead_fwd): z = h W^T
on the tensor cores reduced in the epilogue to lse / H / log pi(y) / ell /
dell -- the theta_old "old log-prob" pass whose entropies give the
high-entropy step mask.  With that mask and
normaliser fixed, the update pass at theta is

    per chunk of whole trajectories (default: the whole shard):
      dart_lmhead_fwd      forward at theta: lse_t, dell_t  (at theta =
                           theta_old the old pass's own DartLoss already
                           holds them: forward_lmhead -> select ->
                           backward_lmhead on one object)
      dart_lmhead_bwd      loss + statistics; the KEPT rows gathered; z of
                           those rows recomputed on the tensor cores and
                           turned into bf16 dz = dL/dz in the TMEM epilogue
      dh[kept] = dz W      the model's backward through the head: two plain
      dW (+)= dz^T h_kept  library GEMMs (cuBLAS via torch.mm, fp32 output)

The [T, V] logits never exist (neither fp32 nor bf16); the only [*, V]
buffer is dz itself, for the kept rows only (rows of masked steps have no
gradient), and the two backward GEMMs run over the kept rows
only.  This module sequences the ABI calls and owns the buffers; the loss
arithmetic runs in the CUDA library.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import numpy as np
import torch

from . import dart
from .dart import Shard


def chunk_shard(layout, shard: Shard, max_rows: int) -> List[Shard]:
    """Greedy split of the shard's trajectories into contiguous ranges with at
    most `max_rows` token rows each (a longer trajectory gets its own chunk)."""
    tso = np.asarray(layout.traj_step_off, dtype=np.int64)
    sto = np.asarray(layout.step_tok_off, dtype=np.int64)
    out = []
    a = shard.traj_begin
    while a < shard.traj_end:
        b = a + 1
        while b < shard.traj_end and sto[tso[b + 1]] - sto[tso[a]] <= max_rows:
            b += 1
        s0, s1 = int(tso[a]), int(tso[b])
        out.append(Shard(a, b, s0, s1, int(sto[s0]), int(sto[s1])))
        a = b
    return out


def _mm_f32(a, b):
    """a @ b with fp32 output from bf16 operands (cuBLAS, fp32 accumulation)."""
    try:
        return torch.mm(a, b, out_dtype=torch.float32)
    except (TypeError, RuntimeError):      # torch without mm(out_dtype=): bf16 output, widened
        return torch.mm(a, b).float()


def backward_grads(dz, hidden_kept, kept_rows, n_kept, weight, dh, dW=None, accumulate=False):
    """The model's backward through the head after dart_lmhead_bwd: two plain
    library GEMMs over the K kept rows (K read back from the device: the host
    needs it for the GEMM shapes).  dh [rows, d] fp32 receives dz W on the
    kept rows (other rows untouched: the caller zeroes them); dW = dz^T
    hidden_kept (added to dW when accumulate).  Returns (dW, K)."""
    K = int(n_kept.item())
    if K == 0:
        if dW is not None and not accumulate:
            dW.zero_()
        return dW, 0
    dzc, hk = dz[:K], hidden_kept[:K]
    dh.index_copy_(0, kept_rows[:K].long(), _mm_f32(dzc, weight))
    g = _mm_f32(dzc.t(), hk)
    if dW is None:
        return g, K
    if accumulate:
        dW.add_(g)
    else:
        dW.copy_(g)
    return dW, K


class LmHeadUpdate:
    """Buffers + ABI sequence of the LM-head update pass for one shard."""

    def __init__(self, layout, V: int, d: int, cfg: dart.Config, device, shard: Optional[Shard] = None,
                 chunk_rows: Optional[int] = None):
        if V % 8 or d % 8:
            raise dart.DartError("the LM-head update needs V % 8 == 0 and d % 8 == 0")
        dev = torch.device(device)
        self.device, self.layout, self.V, self.d = dev, layout, int(V), int(d)
        self.shard = shard or dart.whole_shard(layout)
        self.chunks = chunk_shard(layout, self.shard, chunk_rows) if chunk_rows else [self.shard]
        self.cfg = dataclasses.replace(cfg, stats_accumulate=1)      # chunks add into one stats buffer
        world = list(self.chunks)
        if self.chunks != [dart.whole_shard(layout)]:
            # chunks are virtual ranks of the batch; the shard's other ranks pad the list
            world = [Shard(0, self.shard.traj_begin, 0, self.shard.step_begin, 0, self.shard.tok_begin)] \
                if self.shard.tok_begin > 0 else []
            world += list(self.chunks)
            if self.shard.tok_end < layout.T:
                world.append(Shard(self.shard.traj_end, layout.N_traj, self.shard.step_end, layout.S,
                                   self.shard.tok_end, layout.T))
        self.parts = [dart.DartLoss(layout, c, V, self.cfg, dev, with_grad=False, group=False,
                                    world_shards=world) for c in self.chunks]
        self.stats = torch.zeros(len(dart.STATS_FIELDS), dtype=torch.float64, device=dev)
        self.status = self.parts[0].status
        for p in self.parts:
            p.stats = self.stats               # one accumulator (cfg.stats_accumulate)
            p.status = self.status
        rows = max(c.T_loc for c in self.chunks)
        self.rows = rows
        self.dz = torch.empty((rows, self.V), dtype=torch.bfloat16, device=dev)     # compact kept rows
        self.h_kept = torch.empty((rows, self.d), dtype=torch.bfloat16, device=dev)
        self.kept_rows = torch.empty(rows, dtype=torch.int32, device=dev)
        self.n_kept = torch.zeros(1, dtype=torch.int64, device=dev)
        self.launches = 0
        self.last_n_kept = None

    def run(self, hidden, weight, target, logp_old, logp_roll, logp_ref, keep, norm, dh=None, dW=None):
        """hidden [T_loc, d] bf16, weight [V, d] bf16 (row-major), per-token
        inputs [T_loc], keep [S] / norm from the old-policy pass.  Returns
        (dh [T_loc, d] fp32, dW [V, d] fp32).  (At theta = theta_old the
        old pass's own DartLoss can skip the second forward: forward_lmhead ->
        select -> backward_lmhead on one object, see backward_grads.)"""
        dart._require_cuda(hidden, weight, target, logp_old, logp_roll, logp_ref, keep, norm)
        T = self.shard.T_loc
        if hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16 or hidden.shape != (T, self.d) \
                or weight.shape != (self.V, self.d):
            raise dart.DartError(f"hidden [{T}, {self.d}] / weight [{self.V}, {self.d}] bf16 expected")
        dart._check_token_inputs(self.cfg, T, target, logp_old, logp_roll, logp_ref)
        if keep.dtype != torch.uint8 or not keep.is_contiguous() or keep.numel() < self.layout.S:
            raise dart.DartError(f"keep must be a contiguous uint8 [{self.layout.S}] tensor")
        if norm.dtype != torch.int64 or not norm.is_contiguous() or norm.numel() != 5:
            raise dart.DartError("norm must be the int64 [5] dart_norm of the old-policy pass")
        dh = torch.zeros((T, self.d), dtype=torch.float32, device=self.device) if dh is None else dh.zero_()
        self.stats.zero_()
        n_total = 0
        for i, (c, p) in enumerate(zip(self.chunks, self.parts)):
            r0, r1 = c.tok_begin - self.shard.tok_begin, c.tok_end - self.shard.tok_begin
            hc = hidden[r0:r1]
            p.forward_lmhead(hc, weight, target[r0:r1], logp_old[r0:r1], logp_roll[r0:r1], logp_ref[r0:r1])
            p.backward_lmhead(self.dz, self.h_kept, self.kept_rows, self.n_kept, keep=keep, norm=norm)
            self.launches += p.launches
            p.launches = 0
            dW, K = backward_grads(self.dz, self.h_kept, self.kept_rows, self.n_kept, weight, dh[r0:r1], dW,
                                   accumulate=i > 0)
            n_total += K
        if dW is None:
            dW = torch.zeros((self.V, self.d), dtype=torch.float32, device=self.device)
        self.last_n_kept = n_total
        return dh, dW

    def stats_dict(self):
        return dict(zip(dart.STATS_FIELDS, self.stats.cpu().tolist()))

    def check_status(self):
        v = int(self.status.item())
        if v:
            names = [n for bit, n in dart.STATUS_BITS.items() if v & bit]
            raise dart.DartError(f"DART device status 0x{v:x}: {', '.join(names)}")
