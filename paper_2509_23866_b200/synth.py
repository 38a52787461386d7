"""Seeded synthetic DART training batches -- inputs only.

This module is the one piece shared by the oracle side (tests) and the CUDA
side (tests, bench): it draws random numbers and lays them out.  It holds none
of the method's arithmetic (no advantage, entropy, selection, IS weight or
loss).  The only library call with a "log-softmax" in it is the realism
helper `_approx_target_logp`, which turns the synthetic logits into a
plausible pi_old^Train(y) so that the importance ratios sit near 1 the way a
real trainer's do (DESIGN.md §5 "input recipe"); both sides then receive the
same numbers as plain inputs.

Recipe:
  * steps are routine (70%) or fork (30%) -- most GUI tokens are low-entropy,
    a minority are decision "forks";
  * token row z_v = sigma * eps_v + b * [v == v*], eps ~ N(0,1), v* uniform;
    routine: sigma = 1, b ~ U[17, 30];  fork: sigma ~ U[1, 4] per step,
    b ~ U[0, 15];  rounded to bf16 (fp32 for the tiny config);
  * target y ~ softmax(z / T) by Gumbel-max (temperature 1);
  * logp_old = min(logp + N(0, 0.15^2), 0);  logp_rollout = min(logp_old +
    0.97 N(0, 0.02^2) + 0.03 N(0, 1), 0) (rollout/trainer quantisation
    mismatch);  logp_ref = min(logp + N(0, 0.1^2), 0);
  * rewards R_i ~ Bernoulli(p_g), p_g ~ U[0.1, 0.9], 5% of groups forced
    all-equal (sigma_R = 0 path); parity runs may use real rewards U[0, 1]
    (PAPER.md:280).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np
import torch

V_QWEN = 152064      # UI-TARS-1.5-7B / Qwen2.5-VL vocabulary (BASELINE.json configs)


@dataclasses.dataclass
class Layout:
    """Global batch metadata (CSR), the dart_meta of include/dart_loss.h."""
    G: int
    traj_group: np.ndarray      # int32 [N_traj], non-decreasing
    traj_reward: np.ndarray     # float32 [N_traj]
    traj_step_off: np.ndarray   # int64 [N_traj+1]
    step_tok_off: np.ndarray    # int64 [S+1]
    step_fork: np.ndarray       # bool [S] (generator detail: step type)

    @property
    def N_traj(self):
        return len(self.traj_group)

    @property
    def S(self):
        return len(self.step_tok_off) - 1

    @property
    def T(self):
        return int(self.step_tok_off[-1])


@dataclasses.dataclass
class Batch:
    layout: Layout
    V: int
    logits: torch.Tensor        # [T, V] bf16 or fp32
    target: torch.Tensor        # int32 [T]
    logp_old: torch.Tensor      # fp32 [T]
    logp_rollout: torch.Tensor  # fp32 [T]
    logp_ref: torch.Tensor      # fp32 [T]
    name: str = ""
    logits_store: Optional[torch.Tensor] = None   # [T, ld] storage of `logits` (padded rows)
    ref_logits: Optional[torch.Tensor] = None     # [T, V] reference-policy logits (exact-KL mode)

    def oracle_dict(self, rows=None, logits=True):
        """numpy float64 view for the oracle (exact conversion from bf16/fp32)."""
        L = self.layout
        d = dict(G=L.G, traj_group=L.traj_group.copy(), traj_reward=L.traj_reward.astype(np.float64),
                 traj_step_off=L.traj_step_off.copy(), step_tok_off=L.step_tok_off.copy(),
                 target=self.target.cpu().numpy().astype(np.int64),
                 logp_old=self.logp_old.cpu().numpy().astype(np.float64),
                 logp_rollout=self.logp_rollout.cpu().numpy().astype(np.float64),
                 logp_ref=self.logp_ref.cpu().numpy().astype(np.float64))
        if logits:   # float32 holds bf16 exactly; the oracle widens each row to float64
            d["logits"] = self.logits.float().cpu().numpy()
            if self.ref_logits is not None:
                d["ref_logits"] = self.ref_logits.float().cpu().numpy()
        return d


# ---------------------------------------------------------------- layouts
def _layout(groups, step_tokens_fn, reward_fn, rng, fork_frac=0.3):
    """groups: list over groups of lists of trajectory lengths (steps)."""
    traj_group, traj_steps = [], []
    for g, lens in enumerate(groups):
        for L in lens:
            traj_group.append(g)
            traj_steps.append(int(L))
    traj_step_off = np.zeros(len(traj_steps) + 1, dtype=np.int64)
    traj_step_off[1:] = np.cumsum(traj_steps)
    S = int(traj_step_off[-1])
    ntok = np.asarray([step_tokens_fn(rng) for _ in range(S)], dtype=np.int64)
    step_tok_off = np.zeros(S + 1, dtype=np.int64)
    step_tok_off[1:] = np.cumsum(ntok)
    rewards = reward_fn(groups, rng)
    step_fork = rng.random(S) < fork_frac
    return Layout(G=len(groups), traj_group=np.asarray(traj_group, dtype=np.int32),
                  traj_reward=np.asarray(rewards, dtype=np.float32),
                  traj_step_off=traj_step_off, step_tok_off=step_tok_off, step_fork=step_fork)


def bernoulli_rewards(groups, rng, equal_frac=0.05):
    out = []
    for lens in groups:
        n = len(lens)
        if rng.random() < equal_frac:
            v = float(rng.integers(0, 2))
            out += [v] * n
            continue
        p = rng.uniform(0.1, 0.9)
        r = (rng.random(n) < p).astype(np.float64)
        if n >= 2 and r.min() == r.max():       # keep the group informative
            r[rng.integers(0, n)] = 1.0 - r[0]
        out += list(r)
    return out


def real_rewards(groups, rng):
    return list(rng.random(sum(len(l) for l in groups)))


# ---------------------------------------------------------------- curation inputs
def make_curation_inputs(G, seed=0, tok_lo=16, tok_hi=128, max_len=60, pool_max=3):
    """Seeded raw inputs of one curation round (§4.1-4.2 workload,
    no curation arithmetic here): per task a success history (n_success,
    n_total), the historical max successful length (-1 = none), this
    iteration's rollouts as (per-step token counts, reward) with up to
    `max_len` steps, a pool of stored successes and one uniform draw per
    task.  Roughly a third of the tasks are hard (every rollout fails), a
    third easy (success rate above 0.6)."""
    rng = np.random.default_rng(seed * 7919 + 5)
    kind = rng.integers(0, 3, size=G)                 # 0 hard, 1 medium, 2 easy
    p_succ = np.where(kind == 0, 0.0, np.where(kind == 1, rng.uniform(0.2, 0.6, G), rng.uniform(0.65, 1.0, G)))
    n_total = rng.integers(0, 64, size=G)
    n_success = np.asarray([int(rng.binomial(n, p)) for n, p in zip(n_total, p_succ)], dtype=np.int64)
    max_succ = np.where(n_success > 0, rng.integers(3, 70, size=G), -1).astype(np.int32)
    def traj(success):
        L = int(rng.integers(1, max_len + 1))
        return [int(x) for x in rng.integers(tok_lo, tok_hi + 1, size=L)], (1.0 if success else 0.0)
    def rollouts(n, p):
        return [traj(rng.random() < p) for _ in range(int(n))]
    pool = [[traj(True) for _ in range(int(rng.integers(0, pool_max + 1)))] for _ in range(G)]
    draws = rng.random(G)
    return dict(n_success=n_success, n_total=n_total.astype(np.int64), max_success_len=max_succ,
                p_succ=p_succ, make_rollouts=rollouts, pool=pool, pool_draw=draws, rng=rng)


def layout_from_csr(G, traj_group, traj_reward, traj_step_off, step_tok_off, seed=0, fork_frac=0.3):
    """A Layout over given CSR metadata (e.g. a curated batch); only the
    generator's step types are drawn here."""
    rng = np.random.default_rng(seed * 31 + 3)
    S = len(step_tok_off) - 1
    return Layout(G=int(G), traj_group=np.asarray(traj_group, dtype=np.int32),
                  traj_reward=np.asarray(traj_reward, dtype=np.float32),
                  traj_step_off=np.asarray(traj_step_off, dtype=np.int64),
                  step_tok_off=np.asarray(step_tok_off, dtype=np.int64), step_fork=rng.random(S) < fork_frac)


# ---------------------------------------------------------------- configs
# name -> (groups-builder, tokens-per-step builder, V, dtype, is_cap)
def config_layout(name, seed=0, real_reward=False):
    rng = np.random.default_rng(seed * 1000003 + 17)
    rw = real_rewards if real_reward else bernoulli_rewards
    if name == "tiny":          # 1 task, 4 rollouts, 3 steps x 16 tokens
        return _layout([[3, 3, 3, 3]], lambda r: 16, rw, rng), 512, torch.float32, 2.0
    if name == "tiny_ragged":
        return _layout([[1, 3, 2, 3]], lambda r: 16, rw, rng), 512, torch.float32, 2.0
    if name == "small_multi":   # several groups, ragged, small V (parity, many tiles)
        groups = [list(rng.integers(1, 6, size=int(rng.integers(2, 6)))) for _ in range(5)]
        return _layout(groups, lambda r: int(r.integers(1, 40)), rw, rng), 1000, torch.float32, 1.0
    if name == "mid":           # V = 152064 bf16, ~1-3K tokens, ragged
        groups = [list(rng.integers(1, 5, size=4)) for _ in range(2)]
        return _layout(groups, lambda r: int(r.integers(16, 97)), rw, rng), V_QWEN, torch.bfloat16, 1.0
    if name == "single":        # 8 tasks x 8 rollouts x 15 steps x 64 tokens
        return _layout([[15] * 8 for _ in range(8)], lambda r: 64, rw, rng), V_QWEN, torch.bfloat16, 1.0
    if name == "single_ragged":
        groups = [list(rng.integers(1, 16, size=8)) for _ in range(8)]
        return _layout(groups, lambda r: 64, rw, rng), V_QWEN, torch.bfloat16, 1.0
    if name == "long":          # 16 tasks x 8 rollouts x 50 steps x 128 tokens
        return _layout([[50] * 8 for _ in range(16)], lambda r: 128, rw, rng), V_QWEN, torch.bfloat16, 1.0
    if name == "adaptive":      # N_g ~ U{4..32}, cap ~ U{10..50}, L ~ U{1..cap}, n_s ~ U{16..128}
        groups = []
        for _ in range(32):
            n = int(rng.integers(4, 33))
            cap = int(rng.integers(10, 51))
            groups.append(list(rng.integers(1, cap + 1, size=n)))
        return _layout(groups, lambda r: int(r.integers(16, 129)), rw, rng), V_QWEN, torch.bfloat16, 1.0
    if name == "adaptive_mini":  # the adaptive recipe scaled down for whole-batch oracle parity
        groups = []
        for _ in range(6):
            n = int(rng.integers(2, 9))
            cap = int(rng.integers(2, 9))
            groups.append(list(rng.integers(1, cap + 1, size=n)))
        return _layout(groups, lambda r: int(r.integers(4, 41)), rw, rng), 4099, torch.bfloat16, 1.0
    if name.startswith("scale"):  # scale<k>: 2^k tokens in groups of 8 x 16 steps x 64 tokens
        k = int(name[5:])
        G = (1 << k) // (8 * 16 * 64)
        return _layout([[16] * 8 for _ in range(G)], lambda r: 64, rw, rng), V_QWEN, torch.bfloat16, 1.0
    if name.startswith("grid"):   # grid<G>x<N>x<L>x<n>@<V>  (tests)
        spec, V = name[4:].split("@")
        G, N, L, n = (int(x) for x in spec.split("x"))
        return _layout([[L] * N for _ in range(G)], lambda r, n=n: n, rw, rng), int(V), \
            (torch.float32 if int(V) < 4096 else torch.bfloat16), 1.0
    raise KeyError(name)


# ---------------------------------------------------------------- tensors
def _approx_target_logp(z, y, inv_temperature):
    """Realism helper (library log-softmax, fp32): a plausible log pi(y) for
    building logp_old / logp_ref.  Not part of either implementation."""
    return torch.log_softmax(z.float() * inv_temperature, dim=-1).gather(1, y.long()[:, None])[:, 0]


def make_batch(name, seed=0, device="cpu", real_reward=False, chunk_rows=2048,
               inv_temperature=1.0, zero_delta=False, layout=None, V=None, dtype=None,
               pad_ld: Optional[int] = None, with_ref=False, ref_sigma=0.3, logit_scale=1.0):
    """Builds a Batch for config `name` on `device` (seeded; identical bits for
    the same (name, seed, device type)).  logit_scale multiplies the drawn
    logits before rounding (sharper or flatter rows for parity sweeps); the
    targets and the recorded log-probabilities follow the scaled logits."""
    if layout is None:
        layout, V0, dt0, _ = config_layout(name, seed, real_reward)
        V = V or V0
        dtype = dtype or dt0
    T = layout.T
    dev = torch.device(device)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed * 7919 + 1)
    rng = np.random.default_rng(seed * 31 + 5)
    step_of_tok = np.repeat(np.arange(layout.S), np.diff(layout.step_tok_off))
    fork_tok = layout.step_fork[step_of_tok]
    sigma_step = np.where(layout.step_fork, rng.uniform(1.0, 4.0, layout.S), 1.0)
    sigma = sigma_step[step_of_tok].astype(np.float32)
    b = np.where(fork_tok, rng.uniform(0.0, 15.0, T), rng.uniform(17.0, 30.0, T)).astype(np.float32)
    vstar = rng.integers(0, V, T)
    ld = V if pad_ld is None else pad_ld
    logits_store = torch.empty((T, ld), dtype=dtype, device=dev)
    logits = logits_store[:, :V]
    if pad_ld is not None:
        logits_store[:, V:].fill_(float("nan"))      # padding must never be read
    target = torch.empty(T, dtype=torch.int32, device=dev)
    logp = torch.empty(T, dtype=torch.float32, device=dev)
    sig_t = torch.from_numpy(sigma).to(dev)
    b_t = torch.from_numpy(b).to(dev)
    vs_t = torch.from_numpy(vstar).to(dev)
    for r0 in range(0, T, chunk_rows):
        r1 = min(T, r0 + chunk_rows)
        n = r1 - r0
        z = torch.randn((n, V), generator=gen, device=dev, dtype=torch.float32)
        z.mul_(sig_t[r0:r1, None])
        z[torch.arange(n, device=dev), vs_t[r0:r1]] += b_t[r0:r1]
        if logit_scale != 1.0:
            z.mul_(logit_scale)
        zq = z.to(dtype)
        logits[r0:r1] = zq
        u = torch.rand((n, V), generator=gen, device=dev, dtype=torch.float32).clamp_(1e-20, 1.0)
        gumbel = -torch.log(-torch.log(u))
        y = torch.argmax(zq.float() * inv_temperature + gumbel, dim=1)
        target[r0:r1] = y.to(torch.int32)
        logp[r0:r1] = _approx_target_logp(zq, y, inv_temperature)
        del z, zq, u, gumbel
    d_old = torch.from_numpy(rng.normal(0, 0.15, T).astype(np.float32)).to(dev)
    mix = rng.random(T) < 0.03
    d_roll = np.where(mix, rng.normal(0, 1.0, T), rng.normal(0, 0.02, T)).astype(np.float32)
    d_ref = torch.from_numpy(rng.normal(0, 0.1, T).astype(np.float32)).to(dev)
    if zero_delta:
        d_old = torch.zeros_like(d_old)
    logp_old = torch.clamp(logp + d_old, max=0.0)
    logp_roll = torch.clamp(logp_old + torch.from_numpy(d_roll).to(dev), max=0.0)
    logp_ref = torch.clamp(logp + d_ref, max=0.0)
    ref = None
    if with_ref:   # reference policy: the same logits perturbed by N(0, ref_sigma^2), same dtype
        g2 = torch.Generator(device=dev)
        g2.manual_seed(seed * 7919 + 2)
        ref = torch.empty((T, V), dtype=dtype, device=dev)
        for r0 in range(0, T, chunk_rows):
            r1 = min(T, r0 + chunk_rows)
            ref[r0:r1] = (logits[r0:r1].float() + ref_sigma * torch.randn((r1 - r0, V), generator=g2, device=dev)).to(dtype)
    return Batch(layout=layout, V=V, logits=logits, target=target, logp_old=logp_old,
                 logp_rollout=logp_roll, logp_ref=logp_ref, name=name, logits_store=logits_store, ref_logits=ref)


# ---------------------------------------------------------------- LM-head inputs
@dataclasses.dataclass
class LmBatch:
    """Inputs of the LM-head-fused forward: `batch` carries the metadata and the
    per-token inputs (its `logits` is None), plus hidden [T, d] and weight [V, d]."""
    batch: Batch
    hidden: torch.Tensor        # bf16 [T, d]
    weight: torch.Tensor        # bf16 [V, d]


def make_lmhead(name, d, seed=0, device="cpu", V=None, layout=None, exact=False, inv_temperature=1.0,
                chunk_rows=2048):
    """Seeded LM-head inputs with the logit statistics of make_batch's recipe.

    realistic (exact=False): W_v ~ N(0, I/d) so |W_v| ~ 1; h_t = sigma_t eps_t +
      b_t W_{v*_t} with eps ~ N(0, I_d) and (sigma, b, v*) drawn as in
      make_batch (routine vs fork steps); then z_tv = h_t . W_v ~ sigma N(0,1)
      + b [v == v*] (+ O(b / sqrt(d)) cross terms) -- the same peaked/flat
      mix, now produced by a matrix product.  Both operands rounded to bf16.
    exact=True: h in {-2..2}, W in {-4..4}/64 -- every partial sum of h.W is a
      multiple of 1/64 below 2^13 in magnitude, so any fp32 summation order is
      exact and the tensor-core logits equal the float64 ones bit for bit.
    Targets: Gumbel-max on z / T (z from an fp32 matmul of the bf16 operands,
    a realism helper like _approx_target_logp, not part of either side)."""
    if layout is None:
        layout, V0, _, _ = config_layout(name, seed)
        V = V or V0
    T = layout.T
    dev = torch.device(device)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed * 7919 + 11)
    rng = np.random.default_rng(seed * 31 + 17)
    if exact:
        hidden = torch.randint(-2, 3, (T, d), generator=gen, device=dev).to(torch.bfloat16)
        weight = (torch.randint(-4, 5, (V, d), generator=gen, device=dev).float() / 64.0).to(torch.bfloat16)
    else:
        weight = (torch.randn((V, d), generator=gen, device=dev) / float(np.sqrt(d))).to(torch.bfloat16)
        step_of_tok = np.repeat(np.arange(layout.S), np.diff(layout.step_tok_off))
        fork_tok = layout.step_fork[step_of_tok]
        sigma_step = np.where(layout.step_fork, rng.uniform(1.0, 4.0, layout.S), 1.0)
        sigma = torch.from_numpy(sigma_step[step_of_tok].astype(np.float32)).to(dev)
        b = torch.from_numpy(np.where(fork_tok, rng.uniform(0.0, 15.0, T),
                                      rng.uniform(17.0, 30.0, T)).astype(np.float32)).to(dev)
        vstar = torch.from_numpy(rng.integers(0, V, T)).to(dev)
        hidden = torch.empty((T, d), dtype=torch.bfloat16, device=dev)
        for r0 in range(0, T, chunk_rows):
            r1 = min(T, r0 + chunk_rows)
            h = torch.randn((r1 - r0, d), generator=gen, device=dev) * sigma[r0:r1, None]
            h += b[r0:r1, None] * weight[vstar[r0:r1]].float()
            hidden[r0:r1] = h.to(torch.bfloat16)
    target = torch.empty(T, dtype=torch.int32, device=dev)
    logp = torch.empty(T, dtype=torch.float32, device=dev)
    wf = weight.float()
    for r0 in range(0, T, chunk_rows):
        r1 = min(T, r0 + chunk_rows)
        z = hidden[r0:r1].float() @ wf.T
        u = torch.rand(z.shape, generator=gen, device=dev, dtype=torch.float32).clamp_(1e-20, 1.0)
        y = torch.argmax(z * inv_temperature - torch.log(-torch.log(u)), dim=1)
        target[r0:r1] = y.to(torch.int32)
        logp[r0:r1] = _approx_target_logp(z, y, inv_temperature)
        del z, u
    d_old = torch.from_numpy(rng.normal(0, 0.15, T).astype(np.float32)).to(dev)
    mix = rng.random(T) < 0.03
    d_roll = np.where(mix, rng.normal(0, 1.0, T), rng.normal(0, 0.02, T)).astype(np.float32)
    d_ref = torch.from_numpy(rng.normal(0, 0.1, T).astype(np.float32)).to(dev)
    logp_old = torch.clamp(logp + d_old, max=0.0)
    logp_roll = torch.clamp(logp_old + torch.from_numpy(d_roll).to(dev), max=0.0)
    logp_ref = torch.clamp(logp + d_ref, max=0.0)
    bt = Batch(layout=layout, V=V, logits=None, target=target, logp_old=logp_old, logp_rollout=logp_roll,
               logp_ref=logp_ref, name=name)
    return LmBatch(batch=bt, hidden=hidden, weight=weight)
