"""Helpers for the GPU parity tests: run the CUDA path through the C ABI and
compare it with the float64 oracle element by element (tolerances below are
derived in DESIGN.md §4)."""
import math

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
SEL_TOL = 1e-5       # a step within this (relative) of tau may flip vs the oracle


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


def grad_tol(dz_ref, p_ref, g, dg, out_dtype):
    """Error model of dz_v = g (delta_vy - p_v) in fp32 then rounded:
    |dz_gpu - dz_ref| <= 1 ulp of the output format
                       + dg |dz_ref / g|      (dg = bound on |g_gpu - g|: c*invT*(RTOL_TOK|dell| + ATOL_TOK))
                       + |g| P_REL p_v        (fp32 error of p_v)
                       + FTZ floor."""
    ulp = bf16_ulp(dz_ref) if out_dtype == torch.bfloat16 else np.maximum(np.abs(dz_ref), 2.0 ** -126) * 2.0 ** -23
    return ulp + dg * np.abs(dz_ref) / abs(g) + (abs(g) + dg) * P_REL * p_ref + abs(g) * 2.0 ** -125 + 1e-38


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
    for s in diff:   # only steps whose oracle entropy is within SEL_TOL of its group's tau may flip
        g = int(L.traj_group[np.searchsorted(L.traj_step_off, s, side="right") - 1])
        assert abs(ref["step_H"][s] - tau_ref[g]) <= SEL_TOL * max(1.0, abs(tau_ref[g])), (s, ref["step_H"][s], tau_ref[g])

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
        scale = float(np.sum(np.abs(ref["c_tok"] * ref["ell"]))) + 1e-300
        assert abs(st["loss"] - ref["loss"]) <= RTOL_ENT * scale + 1e-12, (st["loss"], ref["loss"])
        rs = ref["stats"]
        for k in ("n_tok", "n_kept_tok", "n_kept_step"):
            assert st[k] == rs[k], k
        for k in ("sum_w", "sum_adv", "sum_adv2", "sum_H", "sum_kl"):
            assert abs(st[k] - rs[k]) <= 1e-5 * (abs(rs[k]) + 1.0), (k, st[k], rs[k])
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
            assert np.all(dz[t] == 0), f"row {t} must be zero"
            continue
        # p_ref for the error model: recover from dz_ref = g (onehot - p)
        p_ref = -dref / g
        p_ref[ob["target"][t]] = 1.0 - dref[ob["target"][t]] / g
        dg = abs(ref["c_tok"][t] * cfgf["inv_temperature"]) * (RTOL_TOK * abs(ref["dell"][t]) + ATOL_TOK)
        tol = grad_tol(dref, np.abs(p_ref), g, dg, dl.grad_dtype)
        err = np.abs(dz[t] - dref)
        bad = np.nonzero(err > tol)[0]
        assert bad.size == 0, (t, bad[:5], dz[t][bad[:5]], dref[bad[:5]], g)
    return ref
