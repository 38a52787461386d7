"""LM-head-fused update pass (training half).

The forward half is `DartLoss.forward_lmhead` (dart_lmhead_fwd): the
theta_old "old log-prob" pass computed from hidden states, whose entropies
give the high-entropy step mask.  With that mask and
normaliser known (as for NEXT #1, `dart_loss_fused`), the update pass needs
dL/dh and dL/dW of the loss through the LM head z = h W^T:

    per chunk of whole trajectories (<= chunk_rows token rows):
      z_c  = h_c W^T                    dart_gemm_bf16, fp32 logits of the chunk only
      loss terms, dz_c (bf16)           dart_loss_fused on the chunk (a virtual rank)
      dh_c = dz_c W                     dart_gemm_bf16 (W read MN-major)
      dW  += dz_c^T h_c                 dart_gemm_bf16 (both operands MN-major, fp32 accumulate)

so the [T, V] logits and gradient never exist beyond one chunk (the chunk
buffers are chunk_rows x V x 6 bytes).  Chunks are contiguous ranges of whole
trajectories -- exactly the "virtual ranks" of the sharded ABI -- so the
per-token values are those of the unchunked pass.

All arithmetic runs in the CUDA library (tcgen05 GEMMs + the fused loss
kernel); this module only sequences the ABI calls and owns the buffers.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional

import numpy as np
import torch

from . import dart
from .dart import DART_BF16, DART_F32, Shard, _check, _ptr


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


class LmHeadUpdate:
    """Buffers + ABI sequence of the LM-head update pass for one shard."""

    def __init__(self, layout, V: int, d: int, cfg: dart.Config, device, shard: Optional[Shard] = None,
                 chunk_rows: int = 8192, dw_group: int = 1):
        """dw_group: chunks whose dz rows are kept together for ONE dW GEMM
        (K = their rows): the fp32 read-modify-write of dW [V, d] runs once
        per group instead of once per chunk, for dw_group x the dz buffer.
        Measured slower on B200 (update pass 191-193 ms with 2 or 4 vs 188
        with 1, same box: the SM clock under the power cap fell), so 1."""
        if V % 8 or d % 8:
            raise dart.DartError("the LM-head update needs V % 8 == 0 and d % 8 == 0")
        self.L = dart.lib()
        dev = torch.device(device)
        self.device, self.layout, self.V, self.d = dev, layout, int(V), int(d)
        self.cfg = dataclasses_replace(cfg, zero_fill_masked=1)   # masked rows of dz must be zero for the GEMMs
        self.shard = shard or dart.whole_shard(layout)
        self.meta = dart.Meta.from_layout(layout, dev)
        self.chunks = chunk_shard(layout, self.shard, chunk_rows)
        self.rows = max(c.T_loc for c in self.chunks)
        self.dw_group = max(1, int(dw_group))
        grp_rows = [sum(c.T_loc for c in self.chunks[i:i + self.dw_group])
                    for i in range(0, len(self.chunks), self.dw_group)]
        f32 = dict(dtype=torch.float32, device=dev)
        self.z = torch.empty((self.rows, self.V), **f32)                          # fp32 logits of one chunk
        self.dz = torch.empty((max(grp_rows), self.V), dtype=torch.bfloat16, device=dev)   # dz of one dW group
        T, S = self.shard.T_loc, self.shard.S_loc
        self.lse, self.logp = torch.empty(T, **f32), torch.empty(T, **f32)
        self.ell, self.dell = torch.empty(T, **f32), torch.empty(T, **f32)
        self.H = torch.empty(1, **f32)                                            # unused by the fused call
        self.step_ell = torch.zeros(max(S, 1), dtype=torch.float64, device=dev)
        self.adv = torch.empty(max(layout.N_traj, 1), **f32)
        self.group_ok = torch.empty(max(layout.G, 1), dtype=torch.uint8, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.stats_all = torch.zeros((len(self.chunks), len(dart.STATS_FIELDS)), dtype=torch.float64, device=dev)
        ws = 0
        for c in self.chunks:
            b = self._batch(c, None, None, None, None, None)
            ws = max(ws, int(self.L.dart_workspace_size(ctypes.byref(b), ctypes.byref(self.meta.c()),
                                                        ctypes.byref(self.cfg.c()))))
        self.ws_bytes = ws
        self.ws = torch.empty(ws, dtype=torch.uint8, device=dev)
        self.launches = 0

    def _batch(self, c: Shard, z, target, lo, lr, lref):
        return dart.dart_batch(_ptr(z), DART_F32, c.T_loc, self.V, self.V, c.tok_begin, c.step_begin, c.S_loc,
                               _ptr(target), _ptr(lo), _ptr(lr), _ptr(lref))

    def _out(self, c: Shard):
        r0 = c.tok_begin - self.shard.tok_begin
        s0 = c.step_begin - self.shard.step_begin
        off = lambda t, i, es: ctypes.c_void_p(t.data_ptr() + i * es)  # noqa: E731
        return dart.dart_fwd_out(off(self.lse, r0, 4), off(self.logp, r0, 4), _ptr(self.H), off(self.ell, r0, 4),
                                 off(self.dell, r0, 4), None, off(self.step_ell, s0, 8), _ptr(self.adv),
                                 _ptr(self.group_ok), _ptr(self.status))

    def run(self, hidden, weight, target, logp_old, logp_roll, logp_ref, keep, norm, dh=None, dW=None,
            accumulate_dW: bool = False):
        """hidden [T_loc, d] bf16, weight [V, d] bf16 (row-major, unit column
        stride), per-token inputs [T_loc], keep [S] / norm from the old-policy
        pass.  Returns (dh [T_loc, d] fp32, dW [V, d] fp32); dW is overwritten
        unless accumulate_dW."""
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
        dh = torch.empty((T, self.d), dtype=torch.float32, device=self.device) if dh is None else dh
        dW = torch.empty((self.V, self.d), dtype=torch.float32, device=self.device) if dW is None else dW
        s = torch.cuda.current_stream(self.device).cuda_stream
        meta, cfg = ctypes.byref(self.meta.c()), ctypes.byref(self.cfg.c())
        beta = self.cfg.beta_kl > 0
        launches = 0
        g0, goff, ngrp = 0, 0, 0      # first row of the current dW group, its dz fill level, dW GEMMs so far
        for i, c in enumerate(self.chunks):
            r0, r1 = c.tok_begin - self.shard.tok_begin, c.tok_end - self.shard.tok_begin
            n = r1 - r0
            if i % self.dw_group == 0:
                g0, goff = r0, 0
            z, dz, hc = self.z[:n], self.dz[goff:goff + n], hidden[r0:r1]
            dart.gemm_bf16(hc, weight, z)                                        # z_c = h_c W^T
            launches += self.L.dart_last_launch_count()
            b = self._batch(c, z, target[r0:r1], logp_old[r0:r1], logp_roll[r0:r1],
                            logp_ref[r0:r1] if beta else None)
            _check(self.L.dart_loss_fused(ctypes.byref(b), meta, cfg, _ptr(keep), _ptr(norm),
                                          ctypes.byref(self._out(c)), _ptr(dz), DART_BF16, self.V,
                                          _ptr(self.stats_all[i]), _ptr(self.ws), self.ws_bytes, ctypes.c_void_p(s)))
            launches += self.L.dart_last_launch_count()
            dart.gemm_bf16(dz, weight, dh[r0:r1], b_mn_major=True)               # dh_c = dz_c W
            launches += self.L.dart_last_launch_count()
            goff += n
            if (i + 1) % self.dw_group == 0 or i + 1 == len(self.chunks):
                mode = dart.GEMM_ACCUM_F32 if (accumulate_dW or ngrp > 0) else dart.GEMM_STORE_F32
                dart.gemm_bf16(self.dz[:goff], hidden[g0:g0 + goff], dW, a_mn_major=True, b_mn_major=True,
                               mode=mode)                                       # dW (+)= dz_g^T h_g
                launches += self.L.dart_last_launch_count()
                ngrp += 1
        self.launches += launches
        return dh, dW

    def stats_dict(self):
        tot = self.stats_all.sum(dim=0).cpu().tolist()
        return dict(zip(dart.STATS_FIELDS, tot))

    def check_status(self):
        v = int(self.status.item())
        if v:
            names = [n for bit, n in dart.STATUS_BITS.items() if v & bit]
            raise dart.DartError(f"DART device status 0x{v:x}: {', '.join(names)}")


def dataclasses_replace(cfg, **kw):
    import dataclasses
    return dataclasses.replace(cfg, **kw)
