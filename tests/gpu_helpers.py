"""Helpers for the GPU parity tests: run the CUDA path through the C ABI and
compare it with the float64 oracle element by element (tolerances below are
derived in DESIGN.md §4)."""
import math
import os

import numpy as np
import torch

from oracle import dart_oracle as O
from paper_2509_23866_b200 import dart

# ---- tolerances (DESIGN.md §4 "parity bar")
RTOL_ENT = 1e-5      # entropies and loss: north_star rel 1e-5 (fp32 accumulation)
ATOL_ENT = 1e-6      # absolute floor for near-one-hot rows
ATOL_LOGP = 1e-5     # log-prob: fp32 scale c2 = invT*log2(e) carries 6e-8 relative
RTOL_TOK = 1e-5      # per-token ell / dell
ATOL_TOK = 2e-6
P_REL = 4e-6         # fp32 error of p_v relative to p_v (lse2 rounding + ex2.approx + fma)
SEL_BAND = 1e-6      # north_star: the mask is bit-exact except steps within 1e-6 of tau (oracle values)
LOG2E = 1.0 / math.log(2.0)


def p_rel_row(z_row, lse_t, inv_temperature):
    """Relative fp32 error bound of p_v = 2^(c2 z_v - lse2) per element
    (DESIGN.md §4): P_REL plus the rounding of the exponent's two large
    terms -- -lse2 stored as fp32 and c2 z_v with c2 = invT log2(e) in fp32,
    each 2^-24 relative -- times ln 2.  For bf16 rows of magnitude ~30 the
    added term is ~3e-6; for 8x sharper rows (|z| ~ 240) ~3e-5."""
    zc = np.abs(np.where(np.isfinite(z_row), z_row, 0.0)) * (inv_temperature * LOG2E)
    return P_REL + math.log(2.0) * 2.0 ** -24 * (abs(lse_t) * LOG2E + zc)


def loss_tol(ref):
    """Loss bar: 1e-5 relative to sum |c_t ell_t| (L can be ~0)
    plus the loss's sensitivity to the fp32 rounding of log pi(y):
    sum_t |c_t dell_t| dlogp_t with dlogp_t = 2^-22 (|lse_t| + |logp_t|) (the
    max and the target logit enter in fp32, each exact to 2^-24 relative of a
    term of size <= |lse| + |logp|).  A loss made of tiny terms (A = 0 and
    logp_ref ~ logp: ell = beta k3 ~ d^2 / 2) inherits that absolute error,
    far above 1e-5 of its own size; for ordinary batches the term is ~1e-6
    of the loss."""
    dlogp = 2.0 ** -22 * (np.abs(ref["lse"]) + np.abs(ref["logp"])) + 1e-9
    return (RTOL_ENT * float(np.sum(np.abs(ref["c_tok"] * ref["ell"])))
            + float(np.sum(np.abs(ref["c_tok"] * ref["dell"]) * dlogp)) + 1e-12)


def zero_g_row_ok(dz_row, c_tok, dell, inv_temperature, out_dtype):
    """A kept row whose oracle g = c dell invT is exactly 0 (e.g. A = 0 and
    logp_ref = logp in float64): the GPU's g is within dg = |c| invT
    (RTOL_TOK |dell| + ATOL_TOK) of 0, so |dz_v| = |g_gpu| |delta - p| <= dg
    (+ the output rounding).  Masked rows (c = 0) must be exactly zero."""
    if c_tok == 0.0:
        return bool(np.all(dz_row == 0))
    dg = abs(c_tok * inv_temperature) * (RTOL_TOK * abs(dell) + ATOL_TOK)
    return bool(np.all(np.abs(dz_row) <= dg * (1.0 + 2.0 ** -7) + 1e-38))


def run_gpu(batch, cfg, grad_dtype=None, device="cuda", logits=None, runs=1):
    dev = torch.device(device)
    gd = grad_dtype or (torch.float32 if batch.logits.dtype == torch.float32 else torch.bfloat16)
    ld = batch.logits.stride(0)
    ldg = ld if gd.itemsize == batch.logits.element_size() else (ld * batch.logits.element_size()) // gd.itemsize
    ldg = max(ldg, -(-batch.V // 8) * 8)
    dl = dart.DartLoss(batch.layout, dart.whole_shard(batch.layout), batch.V, cfg, dev,
                       logits_dtype=batch.logits.dtype, grad_dtype=gd, ld=ld, ldg=ldg)
    # move the (possibly padded) storage so the row pitch survives the copy
    lg = logits if logits is not None else batch.logits_store.to(dev)[:, :batch.V]
    args = (lg, batch.target.to(dev), batch.logp_old.to(dev), batch.logp_rollout.to(dev), batch.logp_ref.to(dev))
    for _ in range(runs):
        dl.status.zero_()
        dl.run(*args)
    torch.cuda.synchronize()
    return dl


def bf16_ulp(x):
    """ulp of bf16 at |x| (8 significant bits); fp32-normal floor."""
    ax = np.maximum(np.abs(x), 2.0 ** -126)
    return 2.0 ** (np.floor(np.log2(ax)) - 7)


def grad_tol(dz_ref, p_ref, g, dg, out_dtype, p_rel=P_REL):
    """Error model of dz_v = g (delta_vy - p_v) in fp32 then rounded:
    |dz_gpu - dz_ref| <= 1 ulp of the output format
                       + dg |dz_ref / g|      (dg = bound on |g_gpu - g|: c*invT*(RTOL_TOK|dell| + ATOL_TOK))
                       + |g| p_rel p_v        (fp32 error of p_v; p_rel_row())
                       + FTZ floor."""
    ulp = bf16_ulp(dz_ref) if out_dtype == torch.bfloat16 else np.maximum(np.abs(dz_ref), 2.0 ** -126) * 2.0 ** -23
    return ulp + dg * np.abs(dz_ref) / abs(g) + (abs(g) + dg) * p_rel * p_ref + abs(g) * 2.0 ** -125 + 1e-38


def oracle_select_on(dl, batch, cfgf):
    """The oracle's selection applied to the GPU's own fp32 step entropies:
    the integer decision taken in the same precision on both sides."""
    L = batch.layout
    H = dl.step_H.cpu().numpy()[:L.S].astype(np.float64)
    return O.select_steps(H, L.traj_group, L.traj_step_off, dl.group_ok.cpu().numpy()[:L.G], L.G,
                          cfgf["entropy_q"], cfgf["select_rule"])


def compare(dl, batch, cfg, rows=None, check_all_tokens=True, oracle_rows_only=False):
    """Full parity check.  rows: token rows whose dlogits are compared (all if
    None).  Returns the oracle output for further checks."""
    cfgf = cfg.as_f32()
    L = batch.layout
    T = L.T
    ob = batch.oracle_dict()
    if rows is None:
        rows = list(range(T))
    # --- advantages + group_ok (exact decision, values to fp32)
    A_ref, ok_ref = O.advantages(ob["traj_reward"], ob["traj_group"], ob["traj_step_off"], L.G, cfgf["adv_eps"])
    assert np.array_equal(dl.group_ok.cpu().numpy()[:L.G], ok_ref)
    assert np.allclose(dl.adv.cpu().numpy()[:L.N_traj], A_ref, rtol=1e-6, atol=1e-7)

    # --- selection: GPU == oracle rule applied to GPU step entropies (bit-exact)
    keep_gpu = dl.keep.cpu().numpy()[:L.S]
    keep_same, tau_same = oracle_select_on(dl, batch, cfgf)
    assert np.array_equal(keep_gpu, keep_same), "selection differs from the oracle rule on the same values"
    tau_gpu = dl.tau.cpu().numpy()[:L.G].astype(np.float64)
    ok_t = ~np.isnan(tau_same)
    assert np.array_equal(np.isnan(tau_gpu), ~ok_t)
    if cfgf["select_rule"] == O.SEL_LINEAR:
        assert np.allclose(tau_gpu[ok_t], tau_same[ok_t], rtol=1e-7, atol=0)
    else:
        assert np.array_equal(tau_gpu[ok_t].astype(np.float32), tau_same[ok_t].astype(np.float32))

    # --- oracle with the GPU's mask (differences only at near-ties, checked below)
    ref = O.loss_pass(ob, cfgf, keep_override=keep_gpu, rows=rows)
    keep_ref, tau_ref = O.select_steps(ref["step_H"], L.traj_group, L.traj_step_off, ref["group_ok"], L.G,
                                       cfgf["entropy_q"], cfgf["select_rule"])
    diff = np.nonzero(keep_ref != keep_gpu)[0]
    for s in diff:   # only steps whose oracle entropy is within SEL_BAND (1e-6) of its group's tau may flip
        g = int(L.traj_group[np.searchsorted(L.traj_step_off, s, side="right") - 1])
        assert abs(ref["step_H"][s] - tau_ref[g]) <= SEL_BAND, (s, ref["step_H"][s], tau_ref[g])

    # --- per-token forward outputs
    lse = dl.lse.cpu().numpy()
    H = dl.H.cpu().numpy()
    logp = dl.logp.cpu().numpy()
    ell = dl.ell.cpu().numpy()
    dell = dl.dell.cpu().numpy()
    idx = np.arange(T) if check_all_tokens else np.asarray(rows)
    assert np.all(np.abs(lse[idx] - ref["lse"][idx]) <= RTOL_ENT * np.abs(ref["lse"][idx]) + ATOL_ENT), "lse"
    errH = np.abs(H[idx] - ref["H"][idx])
    assert np.all(errH <= RTOL_ENT * np.abs(ref["H"][idx]) + ATOL_ENT), f"H max err {errH.max()}"
    assert np.all(np.abs(logp[idx] - ref["logp"][idx]) <= ATOL_LOGP), "logp"
    # clip decisions near the boundary may legitimately differ (r within 1e-5 of 1-eps_l / 1+eps_h)
    r = ref["r"][idx]
    near = (np.abs(r - (1 - cfgf["eps_low"])) < 1e-5 * r) | (np.abs(r - (1 + cfgf["eps_high"])) < 1e-5 * r)
    ok = ~near
    near_set = set(int(t) for t in idx[near])
    assert np.all(np.abs(ell[idx][ok] - ref["ell"][idx][ok]) <= RTOL_TOK * np.abs(ref["ell"][idx][ok]) + ATOL_TOK), "ell"
    assert np.all(np.abs(dell[idx][ok] - ref["dell"][idx][ok]) <= RTOL_TOK * np.abs(ref["dell"][idx][ok]) + ATOL_TOK), "dell"

    # --- step entropies
    sH = dl.step_H.cpu().numpy()[:L.S]
    assert np.all(np.abs(sH - ref["step_H"]) <= RTOL_ENT * np.abs(ref["step_H"]) + ATOL_ENT), "step entropy"

    # --- normaliser and loss (same mask on both sides)
    nd = dl.norm_dict()
    n = np.diff(L.step_tok_off)
    assert nd["n_keep_step"] == int(keep_gpu.sum())
    assert nd["n_keep_tok"] == int(n[keep_gpu.astype(bool)].sum())
    st = dl.stats_dict()
    if check_all_tokens:
        assert abs(st["loss"] - ref["loss"]) <= loss_tol(ref), (st["loss"], ref["loss"])
        rs = ref["stats"]
        for k in ("n_tok", "n_kept_tok", "n_kept_step"):
            assert st[k] == rs[k], k
        for k in ("sum_w", "sum_adv2", "sum_kl"):
            assert abs(st[k] - rs[k]) <= 1e-5 * (abs(rs[k]) + 1.0), (k, st[k], rs[k])
        # sum of A over kept tokens: every token of a trajectory carries the same fp32-rounded A,
        # so the error adds coherently -- bound it by 1e-5 sum|A| <= 1e-5 sqrt(n sum A^2) (Cauchy-Schwarz)
        sa_tol = 1e-5 * (math.sqrt(rs["n_kept_tok"] * rs["sum_adv2"]) + 1.0)
        assert abs(st["sum_adv"] - rs["sum_adv"]) <= sa_tol, ("sum_adv", st["sum_adv"], rs["sum_adv"])
        # sum of token entropies: each within RTOL_ENT |H| + ATOL_ENT (H >= 0, so sum |H| = sum H)
        assert abs(st["sum_H"] - rs["sum_H"]) <= RTOL_ENT * abs(rs["sum_H"]) + ATOL_ENT * rs["n_tok"], \
            ("sum_H", st["sum_H"], rs["sum_H"])
        assert abs(st["sum_clip"] - rs["sum_clip"]) <= int(near.sum())
        assert abs(st["sum_trunc"] - rs["sum_trunc"]) <= 1

    # --- gradients
    dz = dl.dlogits.float().cpu().numpy()
    V = batch.V
    for t in rows:
        if int(t) in near_set:
            continue
        g = ref["c_tok"][t] * ref["dell"][t] * cfgf["inv_temperature"]
        dref = ref["dz"][t]
        if g == 0.0:
            assert zero_g_row_ok(dz[t], ref["c_tok"][t], ref["dell"][t], cfgf["inv_temperature"], dl.grad_dtype), \
                f"row {t}: oracle g = 0"
            continue
        # p_ref for the error model: recover from dz_ref = g (onehot - p)
        p_ref = -dref / g
        p_ref[ob["target"][t]] = 1.0 - dref[ob["target"][t]] / g
        dg = abs(ref["c_tok"][t] * cfgf["inv_temperature"]) * (RTOL_TOK * abs(ref["dell"][t]) + ATOL_TOK)
        tol = grad_tol(dref, np.abs(p_ref), g, dg, dl.grad_dtype,
                       p_rel=p_rel_row(ob["logits"][t], ref["lse"][t], cfgf["inv_temperature"]))
        err = np.abs(dz[t] - dref)
        bad = np.nonzero(err > tol)[0]
        assert bad.size == 0, (t, bad[:5], dz[t][bad[:5]], dref[bad[:5]], g)
    return ref


# ---- multi-rank results as one whole-batch view, so compare() checks them against the oracle
def snapshot(dl, rows=None):
    """Host copies of one rank's (or virtual rank's) results: its per-token and
    per-step rows plus the replicated global values.  rows: global token rows
    whose dlogits are kept (all of the shard's if None)."""
    sh = dl.shard
    c = lambda t: t.detach().cpu().numpy().copy()       # noqa: E731
    if dl.dlogits is None:
        dz = None
    elif rows is None:
        dz = c(dl.dlogits.float())
    else:
        dz = {int(t): c(dl.dlogits[int(t) - sh.tok_begin].float()) for t in rows if sh.tok_begin <= t < sh.tok_end}
    return dict(tok=(sh.tok_begin, sh.tok_end), step=(sh.step_begin, sh.step_end), traj=(sh.traj_begin, sh.traj_end),
                lse=c(dl.lse), H=c(dl.H), logp=c(dl.logp), ell=c(dl.ell), dell=c(dl.dell),
                step_H=c(dl.step_H[:sh.S_loc]), dlogits=dz,
                group_ok=c(dl.group_ok), adv=c(dl.adv), keep=c(dl.keep), tau=c(dl.tau), norm=c(dl.norm),
                stats=c(dl.stats), status=int(dl.status.item()))


class Assembled:
    """compare()-able view of a sharded pass: per-token / per-step arrays
    concatenated in rank order (shards are contiguous and cover the batch);
    the replicated values (group_ok, A, keep, tau, norm) must be bitwise equal
    on every rank and are taken from rank 0; stats are either all-reduced
    already (equal on every rank) or local partials (summed here)."""

    def __init__(self, parts, layout, grad_dtype=torch.bfloat16, stats_reduced=True):
        parts = sorted(parts, key=lambda p: (p["tok"][0], p["tok"][1]))   # empty shards before their successor
        t = 0
        for p in parts:
            assert p["tok"][0] == t, "shards must tile the batch"
            t = p["tok"][1]
            assert p["status"] == 0, hex(p["status"])
        assert t == layout.T
        r0 = parts[0]
        for p in parts[1:]:
            for k in ("group_ok", "adv", "keep", "tau", "norm"):
                assert np.array_equal(p[k], r0[k], equal_nan=(k == "tau")), f"rank-replicated {k} differs"
            if stats_reduced:
                assert np.array_equal(p["stats"], r0["stats"]), "all-reduced stats differ across ranks"
        T = torch.from_numpy
        for k in ("group_ok", "adv", "keep", "tau", "norm"):
            setattr(self, k, T(r0[k]))
        for k in ("lse", "H", "logp", "ell", "dell"):
            setattr(self, k, T(np.concatenate([p[k][:p["tok"][1] - p["tok"][0]] for p in parts])))
        self.step_H = T(np.concatenate([p["step_H"] for p in parts]))
        if isinstance(r0["dlogits"], dict):      # sampled rows only (the rest stay 0, never compared)
            V = next((len(v) for p in parts for v in p["dlogits"].values()), 1)
            dz = np.zeros((layout.T, V), dtype=np.float32)
            for p in parts:
                for t, v in p["dlogits"].items():
                    dz[t] = v
            self.dlogits = T(dz)
        else:
            self.dlogits = T(np.concatenate([p["dlogits"][:p["tok"][1] - p["tok"][0]] for p in parts]))
        self.stats = T(r0["stats"] if stats_reduced else np.sum([p["stats"] for p in parts], axis=0))
        self.grad_dtype = grad_dtype

    def norm_dict(self):
        n = self.norm
        d = {k: int(n[i]) for i, k in enumerate(dart.NORM_FIELDS[:4])}
        d["inv_norm"] = float(n[4:5].view(torch.float64)[0])
        return d

    def stats_dict(self):
        return dict(zip(dart.STATS_FIELDS, self.stats.tolist()))


def stream_snapshot(sp, dz_local, rows=None):
    """snapshot() of one rank's StreamedPass: its chunks' per-token / per-step
    state concatenated (chunks tile the rank's shard in order), dz_local the
    rank's [T_loc, V] gradient as consume() delivered it."""
    sh = sp.shard
    c = lambda t: t.detach().cpu().numpy().copy()       # noqa: E731
    cat = lambda k, n: np.concatenate([c(st[k][:n(ch)]) for ch, st in zip(sp.chunks, sp.state)])  # noqa: E731
    tok = lambda ch: ch.T_loc     # noqa: E731
    if rows is None:
        dz = c(dz_local.float())
    else:
        dz = {int(t): c(dz_local[int(t) - sh.tok_begin].float()) for t in rows if sh.tok_begin <= t < sh.tok_end}
    return dict(tok=(sh.tok_begin, sh.tok_end), step=(sh.step_begin, sh.step_end), traj=(sh.traj_begin, sh.traj_end),
                lse=cat("lse", tok), H=cat("H", tok), logp=cat("logp", tok), ell=cat("ell", tok),
                dell=cat("dell", tok), step_H=cat("step_H", lambda ch: ch.S_loc), dlogits=dz,
                group_ok=c(sp.group_ok), adv=c(sp.adv), keep=c(sp.keep), tau=c(sp.tau), norm=c(sp.norm),
                stats=c(sp.stats), status=int(sp.status.item()))


# ---- whole-batch oracle comparison at full size (every row, on the host cores)
_FO = {}             # fork-inherited state of full_oracle_compare's workers


def _host_row(buf, i, is_bf16):
    """Row i of a shared-memory buffer as float32, numpy only (no torch in the
    forked workers: its OpenMP pool is not fork-safe)."""
    if is_bf16:
        return (buf[i].astype(np.uint32) << 16).view(np.float32)
    return buf[i]


def _fo_work(span):
    """Oracle rows [r0, r1) of the current chunk (shared-memory tensors), one
    at a time in float64, and the GPU's gradient rows checked against them.
    Returns per row (lse, logp, H, ell, dell, w, r, clipped, kl, trunc + 2 near)."""
    base, r0, r1 = span
    S = _FO
    cf, invT = S["cfg"], S["invT"]
    out = np.zeros((r1 - r0, 10))
    bad, worst = [], 0.0
    for i in range(r0, r1):
        t = base + i
        z = _host_row(S["z"], i, S["z_bf16"]).astype(np.float64)
        y = int(S["y"][t])
        lse, logp, H, p = O.token_row(z, y, invT)
        ell, dell, w, r, clipped, kl = O.token_loss(logp, S["lo"][t], S["lr"][t], S["lref"][t], S["A_tok"][t], cf)
        trunc = math.exp(S["lo"][t] - S["lr"][t]) >= cf["is_cap"]
        near = abs(r - (1 - cf["eps_low"])) < 1e-5 * r or abs(r - (1 + cf["eps_high"])) < 1e-5 * r
        out[i - r0] = (lse, logp, H, ell, dell, w, r, float(clipped), kl, float(trunc) + 2.0 * float(near))
        if S["dz"] is None or near:
            continue
        dz = _host_row(S["dz"], i, S["dz_bf16"])
        c = S["c_tok"][t]
        g = c * dell * invT
        if g == 0.0:
            if np.any(dz != 0):
                bad.append(t)
                worst = np.inf
            continue
        onehot = np.zeros_like(p)
        onehot[y] = 1.0
        dref = g * (onehot - p)
        dg = abs(c * invT) * (RTOL_TOK * abs(dell) + ATOL_TOK)
        ratio = float((np.abs(dz - dref) / grad_tol(dref, np.maximum(p, onehot), g, dg, S["gd"])).max())
        worst = max(worst, ratio)
        if ratio > 1.0:
            bad.append(t)
    return r0, out, bad, worst


def full_oracle_compare(dl, batch, cfg, chunk=4096, procs=None, dlogits=None, tol_report=None, mask_given=False,
                        keep=None):
    """compare() for batches too large for one oracle process: every row of
    `batch` (logits may live on the GPU) goes through the float64 oracle on
    all host cores, chunk by chunk through shared memory, and EVERY GPU
    gradient row is checked against it in the workers (dlogits: the GPU's
    [T, V] gradient, default dl.dlogits).  Then, on the whole batch: step
    entropies, advantages, the oracle's own selection (mask bit-exact except
    steps within SEL_BAND of tau), tau, normaliser, loss and statistics.
    mask_given: the pass took its mask as an input (dart_loss_fused): per-token
    values are checked on the kept rows only, and entropies / the selection
    (computed by the pass that made the mask) are not part of this call.
    Returns a dict of error summaries (for the test log)."""
    import multiprocessing as mp
    cf = cfg.as_f32()
    assert cf["ratio_level"] == O.RATIO_TOKEN and cf["kl_mode"] == O.KL_K3, "token ratio / k3 KL only"
    L = batch.layout
    T, V = L.T, batch.V
    invT = cf["inv_temperature"]
    dz_gpu = dl.dlogits if dlogits is None else dlogits
    ob = batch.oracle_dict(logits=False)
    A_traj, ok_ref = O.advantages(ob["traj_reward"], ob["traj_group"], ob["traj_step_off"], L.G, cf["adv_eps"])
    assert np.array_equal(dl.group_ok.cpu().numpy()[:L.G], ok_ref)
    assert np.allclose(dl.adv.cpu().numpy()[:L.N_traj], A_traj, rtol=1e-6, atol=1e-7)
    t_step = O.step_of_token(L.step_tok_off, T)
    A_tok = A_traj[O.traj_of_step(L.traj_step_off, L.S)[t_step]]
    keep_gpu = (dl.keep if keep is None else keep).cpu().numpy()[:L.S]
    c_tok = O.step_weights(keep_gpu, L.step_tok_off, cf["norm_mode"])[t_step]
    ch = min(chunk, max(T, 1))
    zbuf = torch.empty((ch, V), dtype=batch.logits.dtype).share_memory_()
    dbuf = torch.empty((ch, V), dtype=dz_gpu.dtype).share_memory_() if dz_gpu is not None else None
    _FO.clear()
    np_view = lambda t: t.view(torch.int16).numpy().view(np.uint16) if t.dtype == torch.bfloat16 \
        else t.view(torch.float32).numpy()     # noqa: E731  (shares the tensor's shared memory)
    _FO.update(cfg=cf, invT=invT, z=np_view(zbuf), z_bf16=zbuf.dtype == torch.bfloat16,
               dz=np_view(dbuf) if dbuf is not None else None,
               dz_bf16=dbuf is not None and dbuf.dtype == torch.bfloat16, y=ob["target"], lo=ob["logp_old"], lr=ob["logp_rollout"],
               lref=ob["logp_ref"], A_tok=A_tok, c_tok=c_tok, gd=dl.grad_dtype)
    if procs is None:
        procs = max(1, min(len(os.sched_getaffinity(0)), 64))
    res = np.zeros((T, 10))
    bad, worst = [], 0.0
    # workers fork once and read each chunk from the shared-memory buffers (CPU only)
    with mp.get_context("fork").Pool(procs) as pool:
        for c0 in range(0, T, ch):
            c1 = min(T, c0 + ch)
            n = c1 - c0
            zbuf[:n].copy_(batch.logits[c0:c1])
            if dbuf is not None:
                dbuf[:n].copy_(dz_gpu[c0:c1])
            step = max(1, -(-n // (procs * 4)))
            spans = [(c0, a, min(n, a + step)) for a in range(0, n, step)]
            for r0, out, b, w in pool.imap_unordered(_fo_work, spans):
                res[c0 + r0:c0 + r0 + len(out)] = out
                bad += b
                worst = max(worst, w)
    assert not bad, f"{len(bad)} gradient rows outside the error model, e.g. {sorted(bad)[:8]} (worst {worst:.3g})"
    lse_r, logp_r, H_r, ell_r, dell_r, w_r, r_r = (res[:, k] for k in range(7))
    clipped_r = res[:, 7].astype(bool)
    kl_r = res[:, 8]
    trunc_r = (res[:, 9] % 2).astype(bool)
    near = res[:, 9] >= 2
    rep = {}
    # per-token forward values
    kb = keep_gpu.astype(bool)
    rows_chk = kb[t_step] if mask_given else np.ones(T, dtype=bool)
    lse, logp = dl.lse.cpu().numpy()[rows_chk], dl.logp.cpu().numpy()[rows_chk]
    ell, dell = dl.ell.cpu().numpy()[rows_chk], dl.dell.cpu().numpy()[rows_chk]
    assert np.all(np.abs(lse - lse_r[rows_chk]) <= RTOL_ENT * np.abs(lse_r[rows_chk]) + ATOL_ENT), "lse"
    assert np.all(np.abs(logp - logp_r[rows_chk]) <= ATOL_LOGP), "logp"
    ok = ~near[rows_chk]
    er, dr = ell_r[rows_chk][ok], dell_r[rows_chk][ok]
    assert np.all(np.abs(ell[ok] - er) <= RTOL_TOK * np.abs(er) + ATOL_TOK), "ell"
    assert np.all(np.abs(dell[ok] - dr) <= RTOL_TOK * np.abs(dr) + ATOL_TOK), "dell"
    rep.update(max_grad_err_over_tol=worst, near_clip_rows=int(near.sum()), checked_rows=int(rows_chk.sum()))
    if not mask_given:
        _check_entropies_and_selection(dl, L, H_r, ok_ref, keep_gpu, cf, rep)
    # normaliser (integers, exact) and loss with the GPU's mask (= the oracle's when no flip)
    nd = dl.norm_dict() if not mask_given else None
    n = np.diff(L.step_tok_off)
    if nd is not None:
        assert nd["n_keep_step"] == int(kb.sum()) and nd["n_keep_tok"] == int(n[kb].sum())
    st = dl.stats_dict()
    loss_r = float(np.sum(c_tok * ell_r))
    scale = float(np.sum(np.abs(c_tok * ell_r))) + 1e-300
    assert abs(st["loss"] - loss_r) <= RTOL_ENT * scale + 1e-12, (st["loss"], loss_r)
    rep.update(loss=st["loss"], loss_oracle=loss_r, loss_rel_err=abs(st["loss"] - loss_r) / scale)
    kt = kb[t_step]
    assert st["n_tok"] == T and st["n_kept_tok"] == int(kt.sum()) and st["n_kept_step"] == int(kb.sum())
    sums = [("sum_w", w_r[kt].sum()), ("sum_adv", A_tok[kt].sum()), ("sum_adv2", (A_tok[kt] ** 2).sum()),
            ("sum_kl", kl_r[kt].sum())] + ([] if mask_given else [("sum_H", H_r.sum())])
    for k, v in sums:
        assert abs(st[k] - v) <= 1e-5 * (abs(v) + 1.0), (k, st[k], v)
    assert abs(st["sum_clip"] - clipped_r[kt].sum()) <= int(near.sum())
    assert abs(st["sum_trunc"] - trunc_r[kt].sum()) <= 1
    if tol_report is not None:
        tol_report.update(rep)
    return rep


def _check_entropies_and_selection(dl, L, H_r, ok_ref, keep_gpu, cf, rep):
    """Token and step entropies against the oracle, then the oracle's own
    selection on its float64 step entropies: the GPU mask may differ only at
    steps within SEL_BAND of tau; tau within the entropy tolerance."""
    H = dl.H.cpu().numpy()
    eH = np.abs(H - H_r)
    assert np.all(eH <= RTOL_ENT * np.abs(H_r) + ATOL_ENT), f"H max err {eH.max()}"
    # step entropies, the oracle's own selection, tau
    sH_r = O.step_entropy(H_r, L.step_tok_off)
    sH = dl.step_H.cpu().numpy()[:L.S].astype(np.float64)
    esH = np.abs(sH - sH_r)
    assert np.all(esH <= RTOL_ENT * np.abs(sH_r) + ATOL_ENT), "step entropy"
    keep_r, tau_r = O.select_steps(sH_r, L.traj_group, L.traj_step_off, ok_ref, L.G, cf["entropy_q"],
                                   cf["select_rule"])
    g_of_s = L.traj_group[O.traj_of_step(L.traj_step_off, L.S)]
    flips = np.nonzero(keep_r != keep_gpu)[0]
    for s in flips:
        assert abs(sH_r[s] - tau_r[g_of_s[s]]) <= SEL_BAND, ("mask flip outside the 1e-6 band", s, sH_r[s],
                                                             tau_r[g_of_s[s]])
    tau = dl.tau.cpu().numpy()[:L.G].astype(np.float64)
    okt = ~np.isnan(tau_r)
    assert np.array_equal(np.isnan(tau), ~okt)
    assert np.all(np.abs(tau[okt] - tau_r[okt]) <= RTOL_ENT * np.abs(tau_r[okt]) + ATOL_ENT), "tau"
    # the distance of the nearest step to its threshold, and the fp32 error there
    d_tau = np.abs(sH_r - tau_r[g_of_s])
    rep.update(max_err_H=float(eH.max()), max_err_step_H=float(esH.max()), mask_flips=int(flips.size),
               min_gap_to_tau_nonzero=float(d_tau[d_tau > 0].min()) if np.any(d_tau > 0) else None,
               max_err_tau=float(np.max(np.abs(tau[okt] - tau_r[okt]))) if okt.any() else 0.0)
