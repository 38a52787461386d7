"""Host-side DART data curation (§4.1-4.2, second half).

ctypes marshalling for the library's host functions (csrc/dart_curate.cu,
include/dart_loss.h): dynamic rollout counts, per-task trajectory caps and
the batch assembly with experience-pool injection.  The curated batch is the
CSR metadata (dart_meta) of the loss pass.  All arithmetic runs in the C
library; this module only packs lists into arrays and back.
"""
from __future__ import annotations

import ctypes
import dataclasses
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import dart


class dart_curation_cfg(ctypes.Structure):
    _fields_ = [("n_max", ctypes.c_int32), ("n_min", ctypes.c_int32), ("cap_min", ctypes.c_int32),
                ("cap_max", ctypes.c_int32), ("sr_high_permille", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("success_reward", ctypes.c_double)]


class dart_traj_set(ctypes.Structure):
    _fields_ = [("n_groups", ctypes.c_int64), ("group_off", ctypes.c_void_p), ("traj_step_off", ctypes.c_void_p),
                ("step_tokens", ctypes.c_void_p), ("reward", ctypes.c_void_p)]


class dart_curated(ctypes.Structure):
    _fields_ = [("cap_traj", ctypes.c_int64), ("cap_steps", ctypes.c_int64), ("traj_group", ctypes.c_void_p),
                ("traj_reward", ctypes.c_void_p), ("traj_source", ctypes.c_void_p),
                ("traj_step_off", ctypes.c_void_p), ("step_tok_off", ctypes.c_void_p),
                ("G", ctypes.c_int64), ("N_traj", ctypes.c_int64), ("S", ctypes.c_int64), ("T", ctypes.c_int64)]


@dataclasses.dataclass
class CurationConfig:
    """Paper values and the readings of DESIGN.md §3 R15-R17."""
    n_max: int = 8
    n_min: int = 2
    cap_min: int = 10
    cap_max: int = 50
    sr_high_permille: int = 600
    success_reward: float = 0.5

    def c(self):
        return dart_curation_cfg(self.n_max, self.n_min, self.cap_min, self.cap_max, self.sr_high_permille, 0,
                                 self.success_reward)


# a trajectory = (per-step token counts, reward); a set = list over tasks of lists of trajectories
Trajectory = Tuple[Sequence[int], float]


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a.size else ctypes.c_void_p(0)


class _Set:
    """A list-of-tasks trajectory set packed as the dart_traj_set CSR (arrays kept alive)."""

    def __init__(self, tasks: Sequence[Sequence[Trajectory]]):
        counts = [len(t) for t in tasks]
        self.group_off = np.zeros(len(tasks) + 1, dtype=np.int64)
        self.group_off[1:] = np.cumsum(counts)
        trajs = [tr for t in tasks for tr in t]
        self.traj_step_off = np.zeros(len(trajs) + 1, dtype=np.int64)
        self.traj_step_off[1:] = np.cumsum([len(s) for s, _ in trajs]) if trajs else []
        self.step_tokens = np.asarray([n for s, _ in trajs for n in s], dtype=np.int32)
        self.reward = np.asarray([r for _, r in trajs], dtype=np.float32)
        self.c = dart_traj_set(len(tasks), _ptr(self.group_off), _ptr(self.traj_step_off), _ptr(self.step_tokens),
                               _ptr(self.reward))
        self.n_traj, self.n_steps = len(trajs), int(self.traj_step_off[-1])


def rollout_counts(cfg: CurationConfig, n_success, n_total) -> np.ndarray:
    """dart_rollout_counts: rollouts per task from its success history."""
    ns = np.ascontiguousarray(n_success, dtype=np.int64)
    nt = np.ascontiguousarray(n_total, dtype=np.int64)
    out = np.zeros(len(ns), dtype=np.int32)
    c = cfg.c()
    dart._check(dart.lib().dart_rollout_counts(ctypes.byref(c), ctypes.c_int64(len(ns)), _ptr(ns), _ptr(nt),
                                               _ptr(out)))
    return out


def trajectory_caps(cfg: CurationConfig, max_success_len) -> np.ndarray:
    """dart_trajectory_caps: per-task step caps; -1 = no successful completion yet."""
    ml = np.ascontiguousarray(max_success_len, dtype=np.int32)
    out = np.zeros(len(ml), dtype=np.int32)
    c = cfg.c()
    dart._check(dart.lib().dart_trajectory_caps(ctypes.byref(c), ctypes.c_int64(len(ml)), _ptr(ml), _ptr(out)))
    return out


@dataclasses.dataclass
class CuratedBatch:
    G: int
    traj_group: np.ndarray      # int32 [N]
    traj_reward: np.ndarray     # float32 [N]
    traj_source: np.ndarray     # int64 [N]: rollout index >= 0, or -(pool index + 1)
    traj_step_off: np.ndarray   # int64 [N + 1]
    step_tok_off: np.ndarray    # int64 [S + 1]

    @property
    def N_traj(self):
        return len(self.traj_group)

    @property
    def S(self):
        return len(self.step_tok_off) - 1

    @property
    def T(self):
        return int(self.step_tok_off[-1])


def curate_batch(cfg: CurationConfig, rollouts: Sequence[Sequence[Trajectory]], caps,
                 pool: Optional[Sequence[Sequence[Trajectory]]] = None, pool_draw=None) -> CuratedBatch:
    """dart_curate_batch: caps, pool injection, CSR layout."""
    R = _Set(rollouts)
    P = _Set(pool) if pool is not None else None
    caps_a = np.ascontiguousarray(caps, dtype=np.int32)
    draws = np.ascontiguousarray(pool_draw if pool_draw is not None else np.zeros(len(rollouts)), dtype=np.float64)
    cap_traj = R.n_traj + len(rollouts)
    cap_steps = R.n_steps + (P.n_steps if P else 0)
    tg = np.zeros(max(cap_traj, 1), dtype=np.int32)
    tr = np.zeros(max(cap_traj, 1), dtype=np.float32)
    ts = np.zeros(max(cap_traj, 1), dtype=np.int64)
    tso = np.zeros(cap_traj + 1, dtype=np.int64)
    sto = np.zeros(cap_steps + 1, dtype=np.int64)
    out = dart_curated(cap_traj, cap_steps, _ptr(tg), _ptr(tr), _ptr(ts), _ptr(tso), _ptr(sto), 0, 0, 0, 0)
    c = cfg.c()
    dart._check(dart.lib().dart_curate_batch(ctypes.byref(c), ctypes.byref(R.c), _ptr(caps_a),
                                             ctypes.byref(P.c) if P else None, _ptr(draws), ctypes.byref(out)))
    N, S = int(out.N_traj), int(out.S)
    return CuratedBatch(int(out.G), tg[:N].copy(), tr[:N].copy(), ts[:N].copy(), tso[:N + 1].copy(),
                        sto[:S + 1].copy())
