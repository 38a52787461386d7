"""Thin ctypes binding of libdart_loss.so (include/dart_loss.h).

Argument marshalling only: every step of the DART loss pass runs in the CUDA
library.  PyTorch supplies device memory, the stream and (for N > 1 ranks)
the two collectives between the ABI calls:

    dart_loss_fwd -> all_gather(step entropies) -> dart_select_steps
                  -> dart_loss_bwd -> all_reduce(stats)

There is no CPU fallback: importing this module without the built library, or
calling it on tensors that are not on a CUDA device, raises.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
from typing import Optional

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DART_LIB_PATH") or os.path.join(_HERE, "libdart_loss.so")   # override: tuning builds

# enums (include/dart_loss.h)
DART_OK, DART_ERR_INVALID_ARG, DART_ERR_UNSUPPORTED, DART_ERR_CUDA, DART_ERR_WORKSPACE = range(5)
DART_BF16, DART_F32 = 0, 1
NORM_TOKEN_MEAN_KEPT, NORM_STEP_MEAN_KEPT, NORM_TOKEN_MEAN_ALL, NORM_STEP_MEAN_ALL, NORM_SUM = range(5)
SEL_FLOOR, SEL_CEIL, SEL_LINEAR, SEL_OFF = range(4)
STATUS_BITS = {
    1 << 0: "NONFINITE_LOGIT", 1 << 1: "TARGET_RANGE", 1 << 2: "ROW_ALL_NEGINF",
    1 << 3: "NONFINITE_LOGP", 1 << 4: "EMPTY", 1 << 5: "BAD_CSR", 1 << 6: "TARGET_NEGINF",
    1 << 7: "NONFINITE_LOSS",
}
ABI_VERSION = 6
RATIO_TOKEN, RATIO_STEP = 0, 1
KL_K3, KL_EXACT = 0, 1


class dart_cfg(ctypes.Structure):
    _fields_ = [("eps_low", ctypes.c_float), ("eps_high", ctypes.c_float), ("is_cap", ctypes.c_float),
                ("beta_kl", ctypes.c_float), ("entropy_q", ctypes.c_float),
                ("inv_temperature", ctypes.c_float), ("adv_eps", ctypes.c_float),
                ("norm_mode", ctypes.c_int32), ("select_rule", ctypes.c_int32),
                ("zero_fill_masked", ctypes.c_int32), ("ratio_level", ctypes.c_int32),
                ("kl_mode", ctypes.c_int32), ("stats_accumulate", ctypes.c_int32)]


class dart_meta(ctypes.Structure):
    _fields_ = [("G", ctypes.c_int64), ("N_traj", ctypes.c_int64), ("S", ctypes.c_int64),
                ("T", ctypes.c_int64), ("traj_group", ctypes.c_void_p), ("traj_reward", ctypes.c_void_p),
                ("traj_step_off", ctypes.c_void_p), ("step_tok_off", ctypes.c_void_p)]


class dart_batch(ctypes.Structure):
    _fields_ = [("logits", ctypes.c_void_p), ("logits_dtype", ctypes.c_int32), ("T_loc", ctypes.c_int64),
                ("V", ctypes.c_int64), ("ld", ctypes.c_int64), ("tok_begin", ctypes.c_int64),
                ("step_begin", ctypes.c_int64), ("S_loc", ctypes.c_int64), ("target", ctypes.c_void_p),
                ("logp_old", ctypes.c_void_p), ("logp_rollout", ctypes.c_void_p),
                ("logp_ref", ctypes.c_void_p), ("ref_logits", ctypes.c_void_p), ("ld_ref", ctypes.c_int64)]


class dart_fwd_out(ctypes.Structure):
    _fields_ = [("lse", ctypes.c_void_p), ("logp", ctypes.c_void_p), ("tok_entropy", ctypes.c_void_p),
                ("ell", ctypes.c_void_p), ("dell", ctypes.c_void_p), ("step_entropy", ctypes.c_void_p),
                ("step_ell", ctypes.c_void_p), ("adv", ctypes.c_void_p), ("group_ok", ctypes.c_void_p),
                ("status", ctypes.c_void_p)]


class dart_lmhead(ctypes.Structure):
    _fields_ = [("hidden", ctypes.c_void_p), ("weight", ctypes.c_void_p), ("d", ctypes.c_int64),
                ("ld_h", ctypes.c_int64), ("ld_w", ctypes.c_int64)]


NORM_FIELDS = ["n_keep_tok", "n_keep_step", "n_tok", "n_step", "inv_norm"]  # 4 x i64 + f64
STATS_FIELDS = ["loss", "n_tok", "n_kept_tok", "n_kept_step", "sum_clip", "sum_trunc", "sum_w",
                "sum_adv", "sum_adv2", "sum_H", "sum_kl"]

_lib = None

EXPORTED = ["dart_workspace_size", "dart_loss_fwd", "dart_select_steps", "dart_loss_bwd", "dart_loss_fused",
            "dart_loss_pass", "dart_lmhead_workspace_size", "dart_lmhead_fwd", "dart_lmhead_bwd",
            "dart_status_str", "dart_abi_version", "dart_last_launch_count", "dart_set_timing_events",
            "dart_rollout_counts", "dart_trajectory_caps", "dart_curate_batch"]


class DartError(RuntimeError):
    pass


def lib():
    """Load libdart_loss.so (fails loudly if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DartError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                        "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    L.dart_workspace_size.restype = ctypes.c_size_t
    L.dart_workspace_size.argtypes = [P(dart_batch), P(dart_meta), P(dart_cfg)]
    L.dart_loss_fwd.restype = ctypes.c_int
    L.dart_loss_fwd.argtypes = [P(dart_batch), P(dart_meta), P(dart_cfg), P(dart_fwd_out), ctypes.c_void_p,
                                ctypes.c_size_t, ctypes.c_void_p]
    L.dart_select_steps.restype = ctypes.c_int
    L.dart_select_steps.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                    P(dart_meta), P(dart_cfg), ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                    ctypes.c_void_p]
    L.dart_loss_bwd.restype = ctypes.c_int
    L.dart_loss_bwd.argtypes = [P(dart_batch), P(dart_meta), P(dart_cfg), P(dart_fwd_out), ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    L.dart_loss_fused.restype = ctypes.c_int
    L.dart_loss_fused.argtypes = [P(dart_batch), P(dart_meta), P(dart_cfg), ctypes.c_void_p, ctypes.c_void_p,
                                  P(dart_fwd_out), ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    L.dart_loss_pass.restype = ctypes.c_int
    L.dart_loss_pass.argtypes = [P(dart_batch), P(dart_meta), P(dart_cfg), P(dart_fwd_out), ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                 ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                 ctypes.c_void_p]
    L.dart_lmhead_workspace_size.restype = ctypes.c_size_t
    L.dart_lmhead_workspace_size.argtypes = [P(dart_lmhead), P(dart_batch), P(dart_meta), P(dart_cfg)]
    L.dart_lmhead_fwd.restype = ctypes.c_int
    L.dart_lmhead_fwd.argtypes = [P(dart_lmhead), P(dart_batch), P(dart_meta), P(dart_cfg), P(dart_fwd_out),
                                  ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    L.dart_lmhead_bwd.restype = ctypes.c_int
    L.dart_lmhead_bwd.argtypes = [P(dart_lmhead), P(dart_batch), P(dart_meta), P(dart_cfg), P(dart_fwd_out),
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                  ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_size_t, ctypes.c_void_p]
    L.dart_status_str.restype = ctypes.c_char_p
    L.dart_status_str.argtypes = [ctypes.c_int]
    L.dart_abi_version.restype = ctypes.c_int32
    L.dart_last_launch_count.restype = ctypes.c_int32
    L.dart_set_timing_events.restype = None
    L.dart_set_timing_events.argtypes = [ctypes.c_void_p] * 4
    # host-side curation (paper_2509_23866_b200/curation.py marshals)
    for n in ("dart_rollout_counts", "dart_trajectory_caps", "dart_curate_batch"):
        getattr(L, n).restype = ctypes.c_int
    if L.dart_abi_version() != ABI_VERSION:
        raise DartError(f"libdart_loss ABI {L.dart_abi_version()} != binding {ABI_VERSION}")
    _lib = L
    return L


def _check(rc):
    if rc != DART_OK:
        raise DartError(lib().dart_status_str(rc).decode())


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise DartError("DART tensors must live on a CUDA device (no CPU fallback)")


def set_timing_events(fwd_begin=None, fwd_end=None, bwd_begin=None, bwd_end=None):
    """Have the library record torch.cuda.Event's around its two sweep kernels
    (None disables).  The events must have been recorded once (created)."""
    ev = [ctypes.c_void_p(e.cuda_event) if e is not None else None for e in (fwd_begin, fwd_end, bwd_begin, bwd_end)]
    lib().dart_set_timing_events(*ev)


def _check_token_inputs(cfg, T, target, logp_old, logp_roll, logp_ref):
    """Per-token inputs: int32 targets and fp32 log-probs, contiguous, [T];
    logp_ref only when the k3 KL term reads it (beta > 0, kl_mode = K3)."""
    req = [("target", target, torch.int32), ("logp_old", logp_old, torch.float32),
           ("logp_rollout", logp_roll, torch.float32)]
    if cfg.beta_kl > 0 and cfg.kl_mode == KL_K3:
        if logp_ref is None:
            raise DartError("beta_kl > 0 with the k3 KL needs logp_ref")
        req.append(("logp_ref", logp_ref, torch.float32))
    for name, t, dt in req:
        if t is None or t.dtype != dt or not t.is_contiguous() or t.numel() != T:
            raise DartError(f"{name} must be a contiguous {dt} [{T}] tensor")


# --------------------------------------------------------------------- config
@dataclasses.dataclass
class Config:
    """Hyper-parameters; defaults are the paper's."""
    eps_low: float = 0.2
    eps_high: float = 0.28
    is_cap: float = 1.0
    beta_kl: float = 0.1
    entropy_q: float = 0.2
    inv_temperature: float = 1.0
    adv_eps: float = 0.0
    norm_mode: int = NORM_TOKEN_MEAN_KEPT
    select_rule: int = SEL_FLOOR
    zero_fill_masked: int = 1
    ratio_level: int = RATIO_TOKEN
    kl_mode: int = KL_K3
    stats_accumulate: int = 0     # 1: bwd calls add into the stats buffer (chunked passes)

    def c(self):
        return dart_cfg(self.eps_low, self.eps_high, self.is_cap, self.beta_kl, self.entropy_q,
                        self.inv_temperature, self.adv_eps, self.norm_mode, self.select_rule,
                        self.zero_fill_masked, self.ratio_level, self.kl_mode, self.stats_accumulate)

    def as_f32(self):
        """The values the library actually sees (float32-rounded), for the oracle."""
        import numpy as np
        d = dataclasses.asdict(self)
        for k in ("eps_low", "eps_high", "is_cap", "beta_kl", "entropy_q", "inv_temperature", "adv_eps"):
            d[k] = float(np.float32(d[k]))
        return d


# --------------------------------------------------------------------- metadata
class Meta:
    """Global batch metadata on the device (replicated on every rank)."""

    def __init__(self, G, traj_group, traj_reward, traj_step_off, step_tok_off, device):
        dev = torch.device(device)
        self.G = int(G)
        self.traj_group = torch.as_tensor(traj_group, dtype=torch.int32).to(dev)
        self.traj_reward = torch.as_tensor(traj_reward, dtype=torch.float32).to(dev)
        self.traj_step_off = torch.as_tensor(traj_step_off, dtype=torch.int64).to(dev)
        self.step_tok_off = torch.as_tensor(step_tok_off, dtype=torch.int64).to(dev)
        self.N_traj = int(self.traj_group.numel())
        self.S = int(self.step_tok_off.numel()) - 1
        self.T = int(step_tok_off[-1]) if len(step_tok_off) else 0
        _require_cuda(self.traj_group)

    @classmethod
    def from_layout(cls, layout, device):
        return cls(layout.G, layout.traj_group, layout.traj_reward, layout.traj_step_off,
                   layout.step_tok_off, device)

    def c(self):
        return dart_meta(self.G, self.N_traj, self.S, self.T, _ptr(self.traj_group), _ptr(self.traj_reward),
                         _ptr(self.traj_step_off), _ptr(self.step_tok_off))


@dataclasses.dataclass
class Shard:
    """Local shard = whole trajectories [traj_begin, traj_end)."""
    traj_begin: int
    traj_end: int
    step_begin: int
    step_end: int
    tok_begin: int
    tok_end: int

    @property
    def T_loc(self):
        return self.tok_end - self.tok_begin

    @property
    def S_loc(self):
        return self.step_end - self.step_begin


def whole_shard(layout):
    return Shard(0, layout.N_traj, 0, layout.S, 0, layout.T)


# --------------------------------------------------------------------- the pass
class DartLoss:
    """Buffers + the three ABI calls for one shard of a batch layout.

    `run()` executes one pass on the current CUDA stream; with a process group
    of size > 1 it issues the step-entropy all-gather between fwd and select
    and the statistics all-reduce after bwd (NCCL over NVLink).
    """

    def __init__(self, layout, shard: Shard, V: int, cfg: Config, device, logits_dtype=torch.bfloat16,
                 grad_dtype=torch.bfloat16, group=None, world_shards=None, ld: Optional[int] = None,
                 ldg: Optional[int] = None, ld_ref: Optional[int] = None, with_grad: bool = True):
        self.L = lib()
        dev = torch.device(device)
        self.device = dev
        self.layout = layout
        self.shard = shard
        self.V = int(V)
        self.ld = int(ld) if ld is not None else self.V
        # default gradient row pitch: V rounded up to 16 bytes (the ABI's row alignment)
        per = 16 // torch.empty((), dtype=grad_dtype).element_size()
        self.ldg = int(ldg) if ldg is not None else -(-self.V // per) * per
        self.ld_ref = int(ld_ref) if ld_ref is not None else self.ld
        self.cfg = cfg
        self.group = group
        self.meta = Meta.from_layout(layout, dev)
        self.logits_dtype = logits_dtype
        self.grad_dtype = grad_dtype
        T, S_loc = shard.T_loc, shard.S_loc
        f32 = dict(dtype=torch.float32, device=dev)
        self.lse = torch.empty(T, **f32)
        self.logp = torch.empty(T, **f32)
        self.H = torch.empty(T, **f32)
        self.ell = torch.empty(T, **f32)
        self.dell = torch.empty(T, **f32)
        self.step_H = torch.empty(max(S_loc, 1), **f32)
        self.step_ell = torch.empty(max(S_loc, 1), dtype=torch.float64, device=dev)
        self.adv = torch.empty(max(layout.N_traj, 1), **f32)
        self.group_ok = torch.empty(max(layout.G, 1), dtype=torch.uint8, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.keep = torch.empty(max(layout.S, 1), dtype=torch.uint8, device=dev)
        self.tau = torch.empty(max(layout.G, 1), **f32)
        self.norm = torch.empty(5, dtype=torch.int64, device=dev)          # dart_norm (40 B)
        self.stats = torch.empty(len(STATS_FIELDS), dtype=torch.float64, device=dev)
        # with_grad=False: a forward-only pass (e.g. the LM-head old-log-prob pass) owns no gradient buffer
        self.dlogits_store = torch.empty((T, self.ldg), dtype=grad_dtype, device=dev) if with_grad else None
        self.dlogits = self.dlogits_store[:, :self.V] if with_grad else None
        # world layout for select (rank r owns global steps [rank_step_off[r], [r+1]))
        if world_shards is None:
            if (shard.tok_begin, shard.tok_end, shard.step_begin, shard.step_end) != (0, layout.T, 0, layout.S):
                # select() would read layout.S gathered entries from an S_loc buffer
                raise DartError("a partial shard needs world_shards (every rank's shard) for the selection")
            world_shards = [shard]
        self.world = len(world_shards)
        self.S_pad = max(max(s.S_loc for s in world_shards), 1)
        if self.world == 1:
            self.S_pad = layout.S
        self.rank_step_off = torch.tensor([s.step_begin for s in world_shards] + [world_shards[-1].step_end],
                                          dtype=torch.int64, device=dev)
        self.gathered = torch.empty(self.world * self.S_pad, **f32) if self.world > 1 else None
        self.step_H_pad = torch.zeros(self.S_pad, **f32) if self.world > 1 else None
        b = self._batch(None, None, None, None, None, None)
        self.ws_bytes = int(self.L.dart_workspace_size(ctypes.byref(b), ctypes.byref(self.meta.c()),
                                                       ctypes.byref(cfg.c())))
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)
        self.launches = 0

    def _batch(self, logits, target, logp_old, logp_roll, logp_ref, ref_logits=None):
        dt = DART_BF16 if self.logits_dtype == torch.bfloat16 else DART_F32
        s = self.shard
        return dart_batch(_ptr(logits), dt, s.T_loc, self.V, self.ld, s.tok_begin, s.step_begin, s.S_loc,
                          _ptr(target), _ptr(logp_old), _ptr(logp_roll), _ptr(logp_ref), _ptr(ref_logits),
                          self.ld_ref)

    def _fwd_out(self):
        return dart_fwd_out(_ptr(self.lse), _ptr(self.logp), _ptr(self.H), _ptr(self.ell), _ptr(self.dell),
                            _ptr(self.step_H), _ptr(self.step_ell), _ptr(self.adv), _ptr(self.group_ok),
                            _ptr(self.status))

    def _check_inputs(self, logits, target, logp_old, logp_roll, logp_ref):
        _require_cuda(logits, target, logp_old, logp_roll, logp_ref)
        if logits.dtype != self.logits_dtype:
            raise DartError(f"logits dtype {logits.dtype} != {self.logits_dtype}")
        if logits.dim() != 2 or logits.shape[0] != self.shard.T_loc or logits.shape[1] != self.V:
            raise DartError(f"logits shape {tuple(logits.shape)} != ({self.shard.T_loc}, {self.V})")
        if logits.stride(1) != 1 or logits.stride(0) != self.ld:
            raise DartError(f"logits must be row-major with row pitch ld={self.ld}")
        _check_token_inputs(self.cfg, self.shard.T_loc, target, logp_old, logp_roll, logp_ref)

    def _check_ref(self, ref_logits):
        if self.cfg.kl_mode == KL_EXACT and self.cfg.beta_kl > 0:
            if ref_logits is None:
                raise DartError("kl_mode=KL_EXACT needs ref_logits (the reference policy's logits)")
            _require_cuda(ref_logits)
            if (ref_logits.dtype != self.logits_dtype or ref_logits.shape != (self.shard.T_loc, self.V)
                    or ref_logits.stride(1) != 1 or ref_logits.stride(0) != self.ld_ref):
                raise DartError("ref_logits must match logits' dtype and shape, row pitch ld_ref")
            return ref_logits
        return None

    def forward(self, logits, target, logp_old, logp_roll, logp_ref=None, ref_logits=None, stream=None):
        self._check_inputs(logits, target, logp_old, logp_roll, logp_ref)
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        use_k3 = self.cfg.beta_kl > 0 and self.cfg.kl_mode == KL_K3
        b = self._batch(logits, target, logp_old, logp_roll, logp_ref if use_k3 else None, self._check_ref(ref_logits))
        self._inputs = (b, logits, target, logp_old, logp_roll, logp_ref)
        _check(self.L.dart_loss_fwd(ctypes.byref(b), ctypes.byref(self.meta.c()), ctypes.byref(self.cfg.c()),
                                    ctypes.byref(self._fwd_out()), _ptr(self.ws), self.ws_bytes,
                                    ctypes.c_void_p(st)))
        self.launches += self.L.dart_last_launch_count()

    def forward_lmhead(self, hidden, weight, target, logp_old, logp_roll, logp_ref=None, stream=None):
        """dart_lmhead_fwd: the forward with z = hidden @ weight.T
        computed on the tensor cores and reduced in place -- no logits tensor.
        hidden [T_loc, d] bf16, weight [V, d] bf16 (row pitch may exceed d; d % 8 == 0).
        Outputs land in the same buffers as forward(); select() may follow."""
        _require_cuda(hidden, weight, target, logp_old, logp_roll, logp_ref)
        T = self.shard.T_loc
        if hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
            raise DartError("the LM-head path takes bf16 hidden states and weights")
        if hidden.dim() != 2 or weight.dim() != 2 or hidden.shape[0] != T or weight.shape[0] != self.V \
                or hidden.shape[1] != weight.shape[1] or hidden.stride(1) != 1 or weight.stride(1) != 1:
            raise DartError(f"hidden [{T}, d] and weight [{self.V}, d] row-major expected, got "
                            f"{tuple(hidden.shape)} / {tuple(weight.shape)}")
        _check_token_inputs(self.cfg, T, target, logp_old, logp_roll, logp_ref)
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        use_k3 = self.cfg.beta_kl > 0 and self.cfg.kl_mode == KL_K3
        head = dart_lmhead(_ptr(hidden), _ptr(weight), int(hidden.shape[1]), int(hidden.stride(0)),
                           int(weight.stride(0)))
        b = self._batch(None, target, logp_old, logp_roll, logp_ref if use_k3 else None, None)
        need = int(self.L.dart_lmhead_workspace_size(ctypes.byref(head), ctypes.byref(b),
                                                     ctypes.byref(self.meta.c()), ctypes.byref(self.cfg.c())))
        if need > self.ws_bytes:
            self.ws = torch.empty(need, dtype=torch.uint8, device=self.device)
            self.ws_bytes = need
        self._inputs = (b, None, target, logp_old, logp_roll, logp_ref)
        self._head = (head, hidden, weight)
        _check(self.L.dart_lmhead_fwd(ctypes.byref(head), ctypes.byref(b), ctypes.byref(self.meta.c()),
                                      ctypes.byref(self.cfg.c()), ctypes.byref(self._fwd_out()), _ptr(self.ws),
                                      self.ws_bytes, ctypes.c_void_p(st)))
        self.launches += self.L.dart_last_launch_count()

    def backward_lmhead(self, dz, hidden_kept, kept_rows, n_kept, keep=None, norm=None, stream=None):
        """dart_lmhead_bwd after forward_lmhead (training half):
        loss + statistics into self.stats, and for the K kept rows of the
        shard (device count -> n_kept [1] int64): kept_rows[:K] (int32 local
        rows), hidden_kept[:K] = hidden[kept_rows] and dz[:K] = dL/dz of those
        rows in bf16, from z = h W^T recomputed on the tensor cores (the
        logits never exist).  dz [T_loc, >= V] bf16, hidden_kept [T_loc, >= d]
        bf16, kept_rows [T_loc] int32.  keep / norm default to this object's
        (e.g. after select(); the update pass passes the old pass's)."""
        if getattr(self, "_head", None) is None:
            raise DartError("backward_lmhead needs forward_lmhead first (same object, same workspace)")
        head, hidden, weight = self._head
        T = self.shard.T_loc
        _require_cuda(dz, hidden_kept, kept_rows, n_kept)
        if dz.dtype != torch.bfloat16 or dz.dim() != 2 or dz.shape[0] < T or dz.shape[1] < self.V or dz.stride(1) != 1:
            raise DartError(f"dz must be a row-major bf16 [>= {T}, >= {self.V}] tensor")
        if hidden_kept.dtype != torch.bfloat16 or hidden_kept.dim() != 2 or hidden_kept.shape[0] < T \
                or hidden_kept.shape[1] < head.d or hidden_kept.stride(1) != 1:
            raise DartError(f"hidden_kept must be a row-major bf16 [>= {T}, >= {head.d}] tensor")
        if kept_rows.dtype != torch.int32 or kept_rows.numel() < T or not kept_rows.is_contiguous():
            raise DartError(f"kept_rows must be a contiguous int32 [>= {T}] tensor")
        if n_kept.dtype != torch.int64 or n_kept.numel() < 1:
            raise DartError("n_kept must be an int64 [1] tensor")
        keep = self.keep if keep is None else keep
        norm = self.norm if norm is None else norm
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        b = self._inputs[0]
        _check(self.L.dart_lmhead_bwd(ctypes.byref(head), ctypes.byref(b), ctypes.byref(self.meta.c()),
                                      ctypes.byref(self.cfg.c()), ctypes.byref(self._fwd_out()), _ptr(keep),
                                      _ptr(norm), _ptr(dz), dz.stride(0), _ptr(hidden_kept), hidden_kept.stride(0),
                                      _ptr(kept_rows), _ptr(n_kept), _ptr(self.stats), _ptr(self.ws), self.ws_bytes,
                                      ctypes.c_void_p(st)))
        self.launches += self.L.dart_last_launch_count()

    def gather(self):
        """C1: all-gather of the per-rank step entropies (padded to S_pad)."""
        if self.world == 1:
            return
        from . import dist as D
        self.step_H_pad[:self.shard.S_loc].copy_(self.step_H[:self.shard.S_loc])
        D.all_gather_into(self.gathered, self.step_H_pad, group=self.group)

    def set_gathered(self, gathered: torch.Tensor):
        """Provide the all-gathered [world * S_pad] step entropies directly
        (virtual ranks on one device emulate C1 by concatenation)."""
        self.gathered.copy_(gathered)

    def select(self, stream=None):
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        src = self.gathered if self.world > 1 else self.step_H
        _check(self.L.dart_select_steps(_ptr(src), _ptr(self.rank_step_off), self.world, self.S_pad,
                                        ctypes.byref(self.meta.c()), ctypes.byref(self.cfg.c()),
                                        _ptr(self.group_ok), _ptr(self.keep), _ptr(self.tau), _ptr(self.norm),
                                        _ptr(self.ws), self.ws_bytes, ctypes.c_void_p(st)))
        self.launches += self.L.dart_last_launch_count()

    def backward(self, stream=None):
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        b = self._inputs[0]
        gdt = DART_BF16 if self.grad_dtype == torch.bfloat16 else DART_F32
        _check(self.L.dart_loss_bwd(ctypes.byref(b), ctypes.byref(self.meta.c()), ctypes.byref(self.cfg.c()),
                                    ctypes.byref(self._fwd_out()), _ptr(self.keep), _ptr(self.norm),
                                    _ptr(self.dlogits_store), gdt, self.ldg, _ptr(self.stats), _ptr(self.ws),
                                    self.ws_bytes, ctypes.c_void_p(st)))
        self.launches += self.L.dart_last_launch_count()

    def fused(self, logits, target, logp_old, logp_roll, logp_ref=None, keep=None, norm=None, stream=None):
        """single-read loss + gradient with a step mask
        known in advance (default: this object's keep / norm, e.g. from an
        earlier forward + select on the old-policy logits).  One HBM read of
        each kept row instead of two."""
        self._check_inputs(logits, target, logp_old, logp_roll, logp_ref)
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        keep = self.keep if keep is None else keep
        norm = self.norm if norm is None else norm
        b = self._batch(logits, target, logp_old, logp_roll, logp_ref if self.cfg.beta_kl > 0 else None)
        self._inputs = (b, logits, target, logp_old, logp_roll, logp_ref)
        gdt = DART_BF16 if self.grad_dtype == torch.bfloat16 else DART_F32
        _check(self.L.dart_loss_fused(ctypes.byref(b), ctypes.byref(self.meta.c()), ctypes.byref(self.cfg.c()),
                                      _ptr(keep), _ptr(norm), ctypes.byref(self._fwd_out()), _ptr(self.dlogits_store),
                                      gdt, self.ldg, _ptr(self.stats), _ptr(self.ws), self.ws_bytes,
                                      ctypes.c_void_p(st)))
        self.launches += self.L.dart_last_launch_count()
        self.reduce_stats()
        return self.dlogits

    def reduce_stats(self):
        """C2: all-reduce(SUM) of the fp64 loss / statistics partials."""
        if self.world == 1 or self.group is False:
            return
        from . import dist as D
        D.all_reduce(self.stats, group=self.group)

    def capture(self, logits, target, logp_old, logp_roll, logp_ref=None, ref_logits=None):
        """Capture one whole pass over these (device-resident) inputs into a
        CUDA graph; `graph.replay()` then re-runs it with a single launch from
        the host (the buffers it reads and writes are fixed at capture).
        Single-process passes only (the N > 1 collectives stay eager)."""
        if self.world > 1:
            raise DartError("capture() is for single-process passes")
        self.run(logits, target, logp_old, logp_roll, logp_ref, ref_logits)     # warm-up (attributes, tables)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.run(logits, target, logp_old, logp_roll, logp_ref, ref_logits)
        return g

    def run(self, logits, target, logp_old, logp_roll, logp_ref=None, ref_logits=None):
        """One whole pass (fwd -> C1 -> select -> bwd -> C2), stream-ordered."""
        self.forward(logits, target, logp_old, logp_roll, logp_ref, ref_logits)
        self.gather()
        self.select()
        self.backward()
        self.reduce_stats()
        return self.dlogits

    # ----------------------------------------------------------- results
    def check_status(self):
        v = int(self.status.item())
        if v:
            names = [n for bit, n in STATUS_BITS.items() if v & bit]
            raise DartError(f"DART device status 0x{v:x}: {', '.join(names)}")

    def norm_dict(self):
        n = self.norm.cpu()
        d = {k: int(n[i]) for i, k in enumerate(NORM_FIELDS[:4])}
        d["inv_norm"] = float(n[4:5].view(torch.float64)[0])
        return d

    def stats_dict(self):
        s = self.stats.cpu().tolist()
        return dict(zip(STATS_FIELDS, s))
