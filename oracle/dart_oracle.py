"""DART policy-loss oracle: plain, slow, float64 NumPy. TEST INFRASTRUCTURE ONLY.

What it computes
----------------
The per-token policy-loss pass of DART's trainer (arXiv 2509.23866) over policy
logits, written straight from the paper's definitions, one step at a time, in
the paper's order and notation.  Citations are PAPER.md line numbers in
/root/reference (section / equation in parentheses); SURVEY.md §8(c) holds the
readings taken where the paper is silent or ambiguous (Q1..Q17), repeated in
DESIGN.md §3.

Who may use it
--------------
Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs import this module.  The product path (the CUDA
library behind `paper_2509_23866_b200`) never imports, links or executes it,
and this module imports nothing from the product path: the two share no code.

Every numeric step is pinned by `tests/test_oracle_pins.py` against closed
forms, the paper's / SPEC's worked values, brute force, finite differences and
an independent float64 torch-autograd derivation.  No
function here is "parity unpinned".

Conventions
-----------
* All arithmetic in float64.  bf16 / fp32 inputs convert to float64 exactly.
* Logits z: array [T, V]; row t belongs to global token t.
* Metadata is CSR, exactly as the C ABI takes it (include/dart_loss.h):
  traj_group [N_traj] (non-decreasing), traj_reward [N_traj],
  traj_step_off [N_traj+1], step_tok_off [S+1].
* Configuration values (eps, C, q, ...) are used as given; callers pass the
  float32-rounded values the GPU receives so both sides decide the same
  integers (clip branch, selected steps) from the same numbers.
"""
from __future__ import annotations

import math

import numpy as np

# Normalisation modes and selection rules (same integer codes as the C ABI;
# the oracle defines its own copy, it does not import the binding).
NORM_TOKEN_MEAN_KEPT = 0
NORM_STEP_MEAN_KEPT = 1
NORM_TOKEN_MEAN_ALL = 2
NORM_STEP_MEAN_ALL = 3
NORM_SUM = 4

SEL_FLOOR = 0
SEL_CEIL = 1
SEL_LINEAR = 2
SEL_OFF = 3

KL_K3 = 0           # per-token k3 from log pi_ref(y) (default)
KL_EXACT = 1        # exact full-vocabulary KL(pi_theta || pi_ref) from reference logits

RATIO_TOKEN = 0     # r, w per token (default)
RATIO_STEP = 1      # r, w per step on sum_t log pi(y_t) (PAPER.md:124/257 pi(a|h,s))


# --------------------------------------------------------------------------
# Metadata helpers (pure indexing, no method arithmetic)
# --------------------------------------------------------------------------
def group_trajectories(traj_group, G):
    """List, per group g, of the trajectory indices i with traj_group[i] == g."""
    traj_group = np.asarray(traj_group)
    return [np.nonzero(traj_group == g)[0] for g in range(G)]


def traj_of_step(traj_step_off, S):
    """traj index of every step s (steps of traj i are [off[i], off[i+1]))."""
    off = np.asarray(traj_step_off, dtype=np.int64)
    out = np.empty(S, dtype=np.int64)
    for i in range(len(off) - 1):
        out[off[i]:off[i + 1]] = i
    return out


def step_of_token(step_tok_off, T):
    off = np.asarray(step_tok_off, dtype=np.int64)
    out = np.empty(T, dtype=np.int64)
    for s in range(len(off) - 1):
        out[off[s]:off[s + 1]] = s
    return out


# --------------------------------------------------------------------------
# a1. Group-normalised advantage  (§3.3 step group D;
#     PAPER.md:131-137 A = (R_i - Rbar)/sigma_R with Rbar, sigma_R^2 averaged
#     over the |D| steps of D; SURVEY Q8 step-weighted population std, Q9
#     sigma_R = 0 => group skipped)
# --------------------------------------------------------------------------
def advantages(traj_reward, traj_group, traj_step_off, G, adv_eps=0.0):
    """Returns (A [N_traj] float64, group_ok [G] uint8).

    D_g holds one entry (h,s,a,R_i) per *step* of every trajectory i of task g
    (PAPER.md:118), so each trajectory's reward appears L_i times.
    """
    R = np.asarray(traj_reward, dtype=np.float64)
    off = np.asarray(traj_step_off, dtype=np.int64)
    L = off[1:] - off[:-1]
    A = np.zeros(len(R), dtype=np.float64)
    ok = np.zeros(G, dtype=np.uint8)
    for g, trajs in enumerate(group_trajectories(traj_group, G)):
        if len(trajs) == 0:
            continue
        # the rewards of D: R_i repeated once per step of trajectory i
        R_D = np.concatenate([np.full(L[i], R[i]) for i in trajs])
        if R_D.size == 0:
            continue
        R_bar = np.sum(R_D) / R_D.size
        var = np.sum((R_D - R_bar) ** 2) / R_D.size
        sigma = math.sqrt(var)
        if np.all(R_D == R_D[0]):
            # exact arithmetic gives sigma_R = 0 iff all rewards of D are equal;
            # float rounding of R_bar can leave ~1e-17 residue, so decide it exactly
            # -- and R_bar is then R itself (the residue would otherwise become the
            # advantage (R - R_bar) / adv_eps ~ 1e-11 under the adv_eps flag)
            sigma = 0.0
            R_bar = R_D[0]
        if adv_eps > 0.0:                                     # flag, not the paper
            A[trajs] = (R[trajs] - R_bar) / (sigma + adv_eps)
            ok[g] = 1
        elif sigma > 0.0:
            A[trajs] = (R[trajs] - R_bar) / sigma
            ok[g] = 1
        else:                                                 # skip
            A[trajs] = 0.0
            ok[g] = 0
    return A, ok


# --------------------------------------------------------------------------
# a2. Token distribution, log-prob and entropy
#     p_{t,i,v} = pi_theta(v | ...), with sampling temperature
#     1/inv_temperature, natural log.
# --------------------------------------------------------------------------
def log_softmax_row(z_row, inv_temperature=1.0):
    """Plain definition: z' = z/T, lse = log sum_v exp(z'_v), p = exp(z' - lse).

    Max-shifted for float64 range only (an exact identity).  Returns
    (lse, p) with p a float64 vector; -inf logits give p_v = 0.
    """
    zp = np.asarray(z_row, dtype=np.float64) * float(inv_temperature)
    m = np.max(zp)
    if not np.isfinite(m):
        # all -inf (or +inf/NaN present): undefined distribution
        return float("nan"), np.full(zp.shape, np.nan)
    lse = m + math.log(np.sum(np.exp(zp - m)))
    p = np.exp(zp - lse)
    return lse, p


def token_entropy(p):
    """H = - sum_v p_v log p_v with 0 log 0 = 0."""
    p = np.asarray(p, dtype=np.float64)
    nz = p > 0
    return float(-np.sum(p[nz] * np.log(p[nz])))


def token_row(z_row, y, inv_temperature=1.0):
    """lse, log pi(y), H and p for one logit row (PAPER.md:124 pi_theta(a|h,s)
    at token level per SURVEY Q1; PAPER.md:238 entropy)."""
    lse, p = log_softmax_row(z_row, inv_temperature)
    logp = float(z_row[y]) * float(inv_temperature) - lse
    H = token_entropy(p)
    return lse, logp, H, p


# --------------------------------------------------------------------------
# a3. Step entropy  H_t = mean over the step's thought+action tokens
#     (§4.3)
# --------------------------------------------------------------------------
def step_entropy(H_tok, step_tok_off):
    off = np.asarray(step_tok_off, dtype=np.int64)
    H_tok = np.asarray(H_tok, dtype=np.float64)
    S = len(off) - 1
    out = np.empty(S, dtype=np.float64)
    for s in range(S):
        toks = H_tok[off[s]:off[s + 1]]
        out[s] = np.sum(toks) / len(toks)       # empty step: error (len 0)
    return out


# --------------------------------------------------------------------------
# a5. High-entropy step selection  I[H_t >= tau_D^{0.2}]
#     "top 80% high-entropy steps", "at least larger than 20%
#     steps within the group", Eq. 2 indicator (PAPER.md:256,
#     264).  Threshold per task step-group D, rule FLOOR by default
#     (SURVEY Q6); CEIL, LINEAR and OFF are flags.
# --------------------------------------------------------------------------
def threshold(h_group, q, rule=SEL_FLOOR):
    """tau for one group's step entropies (float64 values)."""
    s = np.sort(np.asarray(h_group, dtype=np.float64))      # ascending
    n = len(s)
    q = float(q)
    if rule == SEL_OFF:
        return -math.inf
    if rule == SEL_FLOOR:
        k = int(math.floor(q * n))
        return float(s[min(k, n - 1)])
    if rule == SEL_CEIL:
        k = min(int(math.ceil(q * n)), n - 1)
        return float(s[k])
    if rule == SEL_LINEAR:                # torch.quantile 'linear' reading
        pos = q * (n - 1)
        lo = int(math.floor(pos))
        hi = min(lo + 1, n - 1)
        frac = pos - lo
        return float(s[lo] + frac * (s[hi] - s[lo]))
    raise ValueError(rule)


def select_steps(step_H, traj_group, traj_step_off, group_ok, G, q, rule=SEL_FLOOR):
    """keep [S] uint8 and tau [G] float64.  keep_s = (H_s >= tau_g) and group_ok_g."""
    step_H = np.asarray(step_H, dtype=np.float64)
    off = np.asarray(traj_step_off, dtype=np.int64)
    keep = np.zeros(len(step_H), dtype=np.uint8)
    tau = np.full(G, np.nan)
    for g, trajs in enumerate(group_trajectories(traj_group, G)):
        steps = np.concatenate([np.arange(off[i], off[i + 1]) for i in trajs]) \
            if len(trajs) else np.zeros(0, dtype=np.int64)
        if steps.size == 0:
            continue
        t = threshold(step_H[steps], q, rule)
        tau[g] = t
        if group_ok[g]:
            keep[steps] = (step_H[steps] >= t).astype(np.uint8)
    return keep, tau


# --------------------------------------------------------------------------
# a2 (cont.). Per-token objective terms
# --------------------------------------------------------------------------
def is_weight(logp_old, logp_roll, C):
    """min(pi_old^Train / pi_old^Rollout, C)  (§4.4, Eq. 2)."""
    return min(math.exp(logp_old - logp_roll), C)


def ratio(logp, logp_old):
    """r = pi_theta^Train / pi_old^Train  (Eq. 1), per token."""
    return math.exp(logp - logp_old)


def clip(r, lo, hi):
    return min(max(r, lo), hi)


def surrogate(r, A, eps_low, eps_high):
    """min(r A, clip(r, 1-eps_low, 1+eps_high) A)  (Eq. 1)."""
    return min(r * A, clip(r, 1.0 - eps_low, 1.0 + eps_high) * A)


def surrogate_dlogp(r, A, eps_low, eps_high):
    """d/dlogp of surrogate(): the branch attaining the min carries the gradient
    (SURVEY Q12).  The unclipped branch r*A has derivative A*r (dr/dlogp = r);
    the clipped branch is constant once r is outside [1-eps_low, 1+eps_high]
    and equals r*A inside it, so either way the derivative is A*r when the
    unclipped branch is (weakly) the minimum and 0 otherwise."""
    unclipped_is_min = r * A <= clip(r, 1.0 - eps_low, 1.0 + eps_high) * A
    return A * r if unclipped_is_min else 0.0


def kl_k3(logp, logp_ref):
    """Per-token k3 estimator of D_KL(pi_theta || pi_ref) (the
    estimator is unstated -- SURVEY Q10): e^d - d - 1, d = logp_ref - logp."""
    d = logp_ref - logp
    return math.exp(d) - d - 1.0


def kl_k3_dlogp(logp, logp_ref):
    d = logp_ref - logp
    return -(math.exp(d) - 1.0)        # d(e^d - d - 1)/dd * dd/dlogp, dd/dlogp = -1


def kl_exact_row(z_row, zref_row, inv_temperature=1.0):
    """D_KL(pi_theta || pi_ref) = sum_v p_v (log p_v - log q_v) over the whole
    vocabulary, p = softmax(z/T), q = softmax(z_ref/T).
    Returns (KL, log p - log q) ; terms with p_v = 0 contribute 0."""
    lse, p = log_softmax_row(z_row, inv_temperature)
    lse_r, q = log_softmax_row(zref_row, inv_temperature)
    zp = np.asarray(z_row, dtype=np.float64) * float(inv_temperature)
    zq = np.asarray(zref_row, dtype=np.float64) * float(inv_temperature)
    with np.errstate(invalid="ignore"):
        lpq = (zp - lse) - (zq - lse_r)                # log p_v - log q_v
    nz = p > 0
    return float(np.sum(p[nz] * lpq[nz])), lpq


def lmhead_logits(hidden, weight):
    """Policy logits from the last hidden state, z_{t,v} = sum_k h_{t,k} W_{v,k}
    (the LM head whose softmax is pi_theta(a|h,s) of PAPER.md:124 Eq. 1; the
    fused variant is SURVEY §8(f) #3).  hidden [T, d], weight [V, d] (the
    nn.Linear layout), both converted exactly to float64; the product is the
    plain float64 matrix product -- no blocking, no rounding to bf16 (the fused
    path never materialises bf16 logits, it keeps the fp32 accumulator)."""
    h = np.asarray(hidden, dtype=np.float64)
    W = np.asarray(weight, dtype=np.float64)
    return h @ W.T


def lmhead_grads(dz, hidden, weight):
    """Chain rule through z = h W^T (training half): given
    dL/dz [T, V] (loss_pass's dz rows), dL/dh = dz W  [T, d] and
    dL/dW = dz^T h  [V, d].  Plain float64 matrix products."""
    dz = np.asarray(dz, dtype=np.float64)
    h = np.asarray(hidden, dtype=np.float64)
    W = np.asarray(weight, dtype=np.float64)
    return dz @ W, dz.T @ h


def token_loss(logp, logp_old, logp_roll, logp_ref, A, cfg):
    """ell_t = -w * min(rA, clip(r)A) + beta * KL_k3  -- the library minimises
    L = -J_HE (Eq. 2; SURVEY Q3 the IS weight multiplies the
    surrogate only, Q4 sign).  Returns (ell, dell/dlogp, w, r, clipped, kl)."""
    w = is_weight(logp_old, logp_roll, cfg["is_cap"])
    r = ratio(logp, logp_old)
    sur = surrogate(r, A, cfg["eps_low"], cfg["eps_high"])
    dsur = surrogate_dlogp(r, A, cfg["eps_low"], cfg["eps_high"])
    beta = cfg["beta_kl"]
    kl = kl_k3(logp, logp_ref) if beta != 0.0 else 0.0
    dkl = kl_k3_dlogp(logp, logp_ref) if beta != 0.0 else 0.0
    ell = -w * sur + beta * kl
    dell = -w * dsur + beta * dkl
    clipped = not (r * A <= clip(r, 1.0 - cfg["eps_low"], 1.0 + cfg["eps_high"]) * A)
    return ell, dell, w, r, clipped, kl


# --------------------------------------------------------------------------
# a6. Normalisation of the expectation over D  (PAPER.md:255 E over D; token
#     aggregation unstated -- SURVEY Q11: default token-mean over kept tokens)
# --------------------------------------------------------------------------
def step_weights(keep, step_tok_off, mode, per_step_loss=False):
    """Per-step multiplier c_s so that L = sum_s c_s * sum_{t in s} ell_t.
    per_step_loss: the loss term is already one number per step (step-ratio
    mode), so the step-mean modes drop their 1/n_s factor."""
    off = np.asarray(step_tok_off, dtype=np.int64)
    n = (off[1:] - off[:-1]).astype(np.float64)
    keep = np.asarray(keep).astype(bool)
    S = len(n)
    T = float(np.sum(n))
    c = np.zeros(S, dtype=np.float64)
    if mode == NORM_TOKEN_MEAN_KEPT:
        N = float(np.sum(n[keep]))
        if N > 0:
            c[keep] = 1.0 / N
    elif mode == NORM_STEP_MEAN_KEPT:
        N = float(np.sum(keep))
        if N > 0:
            c[keep] = 1.0 / (N * (1.0 if per_step_loss else n[keep]))
    elif mode == NORM_TOKEN_MEAN_ALL:
        if T > 0:
            c[keep] = 1.0 / T
    elif mode == NORM_STEP_MEAN_ALL:
        if S > 0:
            c[keep] = 1.0 / (S * (1.0 if per_step_loss else n[keep]))
    elif mode == NORM_SUM:
        c[keep] = 1.0
    else:
        raise ValueError(mode)
    return c


# --------------------------------------------------------------------------
# The whole pass
# --------------------------------------------------------------------------
DEFAULT_CFG = dict(eps_low=0.2, eps_high=0.28, is_cap=1.0, beta_kl=0.1,
                   entropy_q=0.2, inv_temperature=1.0, adv_eps=0.0,
                   norm_mode=NORM_TOKEN_MEAN_KEPT, select_rule=SEL_FLOOR,
                   ratio_level=RATIO_TOKEN)
# (PAPER.md:575 eps_low 0.2, eps_high 0.28, beta 0.1, C 1; PAPER.md:578
#  temperature 1.0; PAPER.md:235/264 the 0.2 quantile)


def loss_pass(batch, cfg, keep_override=None, want_grad=True, rows=None):
    """Full DART loss pass on one (global) batch.

    batch: dict with logits [T,V], target [T], logp_old [T], logp_rollout [T],
           logp_ref [T] or None, traj_group, traj_reward, traj_step_off,
           step_tok_off, G.
    keep_override: optional [S] mask replacing step 5's selection (used by the
           parity tests when a step sits within the tolerance of tau).
    rows: optional iterable of token rows for which to return dz (all if None).
    Returns a dict of every intermediate and output, float64.
    """
    cfg = {**DEFAULT_CFG, **cfg}
    z = batch["logits"]
    T, V = z.shape
    y = np.asarray(batch["target"], dtype=np.int64)
    lo = np.asarray(batch["logp_old"], dtype=np.float64)
    lr = np.asarray(batch["logp_rollout"], dtype=np.float64)
    lref = batch.get("logp_ref")
    lref = np.zeros(T) if lref is None else np.asarray(lref, dtype=np.float64)
    G = int(batch["G"])
    traj_step_off = np.asarray(batch["traj_step_off"], dtype=np.int64)
    step_tok_off = np.asarray(batch["step_tok_off"], dtype=np.int64)
    S = len(step_tok_off) - 1
    invT = float(cfg["inv_temperature"])

    # 1. advantages per group
    A_traj, group_ok = advantages(batch["traj_reward"], batch["traj_group"],
                                  traj_step_off, G, cfg["adv_eps"])
    s_traj = traj_of_step(traj_step_off, S)
    t_step = step_of_token(step_tok_off, T)
    A_tok = A_traj[s_traj[t_step]]

    # 2. per token: lse, log-prob, entropy
    lse = np.empty(T)
    logp = np.empty(T)
    H = np.empty(T)
    P = {} if want_grad else None
    want_rows = set(range(T)) if rows is None else set(int(r) for r in rows)
    for t in range(T):
        lse[t], logp[t], H[t], p = token_row(z[t], y[t], invT)
        if want_grad and t in want_rows:
            P[t] = p

    # 3. step entropy
    step_H = step_entropy(H, step_tok_off)

    # 4. selection per group
    keep, tau = select_steps(step_H, batch["traj_group"], traj_step_off,
                             group_ok, G, cfg["entropy_q"], cfg["select_rule"])
    if keep_override is not None:
        keep = np.asarray(keep_override, dtype=np.uint8).copy()

    # 5. per-token objective terms
    ell = np.empty(T)
    dell = np.empty(T)
    w = np.empty(T)
    r = np.empty(T)
    clipped = np.zeros(T, dtype=bool)
    kl = np.empty(T)
    trunc = np.zeros(T, dtype=bool)
    step_ratio = cfg.get("ratio_level", RATIO_TOKEN) == RATIO_STEP
    exact_kl = cfg.get("kl_mode", KL_K3) == KL_EXACT and cfg["beta_kl"] != 0.0
    kl_ex = np.zeros(T)
    LPQ = {}
    if exact_kl:
        zr = batch["ref_logits"]
        for t in range(T):
            kl_ex[t], lpq = kl_exact_row(z[t], zr[t], invT)
            if want_grad and t in want_rows:
                LPQ[t] = lpq
        # the KL term no longer flows through log pi(y): token_loss sees beta = 0
        cfg_tok = {**cfg, "beta_kl": 0.0}
    else:
        cfg_tok = cfg
    if not step_ratio:
        for t in range(T):
            ell[t], dell[t], w[t], r[t], clipped[t], kl[t] = token_loss(
                logp[t], lo[t], lr[t], lref[t], A_tok[t], cfg_tok)
            trunc[t] = math.exp(lo[t] - lr[t]) >= cfg["is_cap"]
            if exact_kl:
                kl[t] = kl_ex[t]
                ell[t] += cfg["beta_kl"] * kl_ex[t]
    else:
        # step-level ratio and IS weight on the step's sequence log-probability
        # log pi(a|h,s) = sum_{t in s} log pi(y_t)
        beta = cfg["beta_kl"]
        for s_ in range(S):
            if exact_kl:
                beta_tok = 0.0
            else:
                beta_tok = beta
            toks = np.arange(step_tok_off[s_], step_tok_off[s_ + 1])
            A_s = A_tok[toks[0]]
            log_r = float(np.sum(logp[toks] - lo[toks]))
            log_w = float(np.sum(lo[toks] - lr[toks]))
            r_s = math.exp(log_r)
            w_s = min(math.exp(log_w), cfg["is_cap"])
            sur = surrogate(r_s, A_s, cfg["eps_low"], cfg["eps_high"])
            dsur = surrogate_dlogp(r_s, A_s, cfg["eps_low"], cfg["eps_high"])   # d/d(log r_s)
            kls = np.array([(kl_ex[t] if exact_kl else kl_k3(logp[t], lref[t])) if beta != 0.0 else 0.0
                            for t in toks])
            ell_s = -w_s * sur + beta * float(np.sum(kls))
            clip_s = not (r_s * A_s <= clip(r_s, 1.0 - cfg["eps_low"], 1.0 + cfg["eps_high"]) * A_s)
            for j, t in enumerate(toks):
                # d ell_s / d logp_t: d log r_s / d logp_t = 1
                dk = kl_k3_dlogp(logp[t], lref[t]) if beta_tok != 0.0 else 0.0
                dell[t] = -w_s * dsur + beta_tok * dk
                ell[t] = ell_s / len(toks)
                w[t], r[t], clipped[t], kl[t] = w_s, r_s, clip_s, kls[j]
                trunc[t] = math.exp(log_w) >= cfg["is_cap"]

    # 6. normalisation and loss
    c_step = step_weights(keep, step_tok_off, cfg["norm_mode"], per_step_loss=step_ratio)
    c_tok = c_step[t_step]
    loss = float(np.sum(c_tok * ell))

    out = dict(A_traj=A_traj, group_ok=group_ok, A_tok=A_tok, lse=lse, logp=logp,
               H=H, step_H=step_H, keep=keep, tau=tau, ell=ell, dell=dell, w=w,
               r=r, clipped=clipped, kl=kl, c_tok=c_tok, loss=loss)

    # statistics (sums; SURVEY §5 metrics)
    kt = keep[t_step].astype(bool)
    n = (step_tok_off[1:] - step_tok_off[:-1])
    out["stats"] = dict(
        loss=loss, n_tok=float(T), n_kept_tok=float(np.sum(n[keep.astype(bool)])),
        n_kept_step=float(np.sum(keep)),
        sum_clip=float(np.sum(clipped[kt])),
        sum_trunc=float(np.sum(trunc[kt])),
        sum_w=float(np.sum(w[kt])), sum_adv=float(np.sum(A_tok[kt])),
        sum_adv2=float(np.sum(A_tok[kt] ** 2)), sum_H=float(np.sum(H)),
        sum_kl=float(np.sum(kl[kt])))

    # 7. gradient w.r.t. logits: dL/dz_{t,v} = c_t * dell_t * invT * (onehot - p)
    if want_grad:
        dz = {}
        for t in sorted(want_rows):
            g = c_tok[t] * dell[t]
            onehot = np.zeros(V)
            onehot[y[t]] = 1.0
            dz[t] = g * invT * (onehot - P[t]) if g != 0.0 else np.zeros(V)
            if exact_kl and c_tok[t] != 0.0:
                # d KL_t / d z_v = invT p_v ((log p_v - log q_v) - KL_t)
                pk = P[t]
                term = np.where(pk > 0, pk * (np.nan_to_num(LPQ[t], nan=0.0, posinf=0.0, neginf=0.0) - kl_ex[t]), 0.0)
                dz[t] = dz[t] + c_tok[t] * cfg["beta_kl"] * invT * term
        out["dz"] = dz
    return out
