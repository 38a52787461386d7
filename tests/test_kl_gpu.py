"""exact full-vocabulary KL(pi_theta || pi_ref) from the
reference policy's logits (DART_KL_EXACT): both sweeps stream z and z_ref.
GPU vs the float64 oracle (its exact-KL path is pinned by the SPEC example,
Gibbs, torch.kl_div, finite differences and autograd)."""
import numpy as np
import pytest
import torch

from oracle import dart_oracle as O
from paper_2509_23866_b200 import dart, synth
from tests.gpu_helpers import ATOL_ENT, ATOL_LOGP, ATOL_TOK, RTOL_ENT, RTOL_TOK, bf16_ulp, oracle_select_on, p_rel_row

pytestmark = pytest.mark.gpu

# Absolute accuracy of one token's exact KL on the GPU: KL_t = sum_v p (z' - z'_ref)
# - (lse - lse_ref) comes from fp32-accumulated sums (flushed to fp64 every 8
# chunks) of terms of size |z' - z'_ref| ~ |lse - lse_ref| + O(1), so it carries
# ~1e-7 absolute error however small KL_t is; a bar relative to
# KL_t alone fails on near-identical policies (KL ~ 1e-8 .. 1e-3 per token).
KL_ATOL = 4e-7


def _run(b, cfg, grad_dtype=None):
    dev = torch.device("cuda")
    gd = grad_dtype or (torch.float32 if b.logits.dtype == torch.float32 else torch.bfloat16)
    dl = dart.DartLoss(b.layout, dart.whole_shard(b.layout), b.V, cfg, dev, logits_dtype=b.logits.dtype,
                       grad_dtype=gd)
    dl.run(b.logits.to(dev), b.target.to(dev), b.logp_old.to(dev), b.logp_rollout.to(dev), b.logp_ref.to(dev),
           ref_logits=b.ref_logits.to(dev))
    torch.cuda.synchronize()
    dl.check_status()
    return dl


def _check(dl, b, cfg, rows, grad_atol=0.0):
    """grad_atol: an absolute floor for the dlogits comparison (the north_star's
    2e-3 on bf16 gradients) -- used for the stress inputs of the path fuzz,
    whose 8x sharper rows and masked vocabularies are outside the per-element
    error model below; 0 keeps the model alone."""
    cfgf = cfg.as_f32()
    L = b.layout
    keep = dl.keep.cpu().numpy()[:L.S]
    keep_same, _ = oracle_select_on(dl, b, cfgf)
    assert np.array_equal(keep, keep_same)
    ob = b.oracle_dict()
    ref = O.loss_pass(ob, cfgf, keep_override=keep, rows=rows)
    H, kl, ell = dl.H.cpu().numpy(), None, dl.ell.cpu().numpy()
    assert np.all(np.abs(H - ref["H"]) <= RTOL_ENT * ref["H"] + ATOL_ENT)
    assert np.all(np.abs(dl.logp.cpu().numpy() - ref["logp"]) <= ATOL_LOGP)
    r = ref["r"]
    ok = ~((np.abs(r - (1 - cfgf["eps_low"])) < 1e-5 * r) | (np.abs(r - (1 + cfgf["eps_high"])) < 1e-5 * r))
    assert np.all(np.abs(ell[ok] - ref["ell"][ok]) <= RTOL_TOK * np.abs(ref["ell"][ok]) + ATOL_TOK)
    st = dl.stats_dict()
    scale = float(np.sum(np.abs(ref["c_tok"] * ref["ell"]))) + 1e-300
    kl_slack = cfgf["beta_kl"] * KL_ATOL * float(np.sum(np.abs(ref["c_tok"])))
    assert abs(st["loss"] - ref["loss"]) <= RTOL_ENT * scale + kl_slack + 1e-12, (st["loss"], ref["loss"])
    n_kept = ref["stats"]["n_kept_tok"]
    assert abs(st["sum_kl"] - ref["stats"]["sum_kl"]) <= 1e-5 * abs(ref["stats"]["sum_kl"]) + KL_ATOL * n_kept + 1e-9, \
        (st["sum_kl"], ref["stats"]["sum_kl"])
    dz = dl.dlogits.float().cpu().numpy()
    invT = cfgf["inv_temperature"]
    for t in rows:
        c = ref["c_tok"][t]
        if c == 0.0:
            assert np.all(dz[t] == 0), t
            continue
        if not ok[t]:
            continue
        _, p = O.log_softmax_row(ob["logits"][t], invT)
        klt, lpq = O.kl_exact_row(ob["logits"][t], ob["ref_logits"][t], invT)
        lpq = np.where(p > 0, np.nan_to_num(lpq, nan=0.0, posinf=0.0, neginf=0.0), 0.0)   # p = 0: no term
        dref = ref["dz"][t]
        # error model: 1 output ulp + dell's tolerance through |delta - p| + the fp32
        # error of p (p_rel_row: grows with the exponent's magnitude) and of
        # (log p - log q) = (z' - z'_ref) - (lse - lse_ref), whose fp32 terms are
        # each exact to 2^-24 of their size (rows of 8x sharper logits reach ~250)
        onehot = np.zeros_like(p)
        onehot[ob["target"][t]] = 1.0
        a = abs(c * invT)
        zf = np.abs(np.where(np.isfinite(ob["logits"][t]), ob["logits"][t], 0.0)).max() * invT
        zrf = np.abs(np.where(np.isfinite(ob["ref_logits"][t]), ob["ref_logits"][t], 0.0)).max() * invT
        lpq_err = 2e-5 + 2.0 ** -21 * (zf + zrf)
        prel = p_rel_row(ob["logits"][t], ref["lse"][t], invT)
        tol = (bf16_ulp(dref) if dl.grad_dtype == torch.bfloat16 else np.abs(dref) * 2.0 ** -22)
        tol = tol + a * (RTOL_TOK * abs(ref["dell"][t]) + ATOL_TOK) * np.abs(onehot - p)
        tol = tol + a * prel * p * (abs(ref["dell"][t]) + cfgf["beta_kl"] * (np.abs(lpq) + klt + 1.0))
        tol = tol + a * cfgf["beta_kl"] * p * lpq_err * (1.0 + np.abs(lpq)) + 1e-38
        tol = np.maximum(tol, grad_atol)
        err = np.abs(dz[t] - dref)
        assert np.all(err <= tol), (t, np.argmax(err - tol), err.max())


@pytest.mark.parametrize("ratio", [dart.RATIO_TOKEN, dart.RATIO_STEP])
@pytest.mark.parametrize("norm", [dart.NORM_TOKEN_MEAN_KEPT, dart.NORM_STEP_MEAN_KEPT])
def test_exact_kl_small(ratio, norm):
    b = synth.make_batch("small_multi", seed=8, with_ref=True)
    cfg = dart.Config(kl_mode=dart.KL_EXACT, beta_kl=0.2, ratio_level=ratio, norm_mode=norm)
    dl = _run(b, cfg)
    _check(dl, b, cfg, rows=list(range(b.layout.T)))


def test_exact_kl_odd_vocab_bf16():
    layout, _, _, _ = synth.config_layout("small_multi", seed=9)
    b = synth.make_batch("small_multi", seed=9, layout=layout, V=1003, dtype=torch.bfloat16, with_ref=True)
    cfg = dart.Config(kl_mode=dart.KL_EXACT)
    # odd V: row pitch must be padded to 16 B for both logits and ref_logits
    dev = torch.device("cuda")
    ld = 1008
    lg = torch.zeros((b.layout.T, ld), dtype=torch.bfloat16, device=dev)[:, :b.V]
    lg.copy_(b.logits)
    rf = torch.zeros((b.layout.T, ld), dtype=torch.bfloat16, device=dev)[:, :b.V]
    rf.copy_(b.ref_logits)
    dl = dart.DartLoss(b.layout, dart.whole_shard(b.layout), b.V, cfg, dev, logits_dtype=torch.bfloat16,
                       grad_dtype=torch.bfloat16, ld=ld, ldg=ld, ld_ref=ld)
    dl.run(lg, b.target.to(dev), b.logp_old.to(dev), b.logp_rollout.to(dev), b.logp_ref.to(dev), ref_logits=rf)
    torch.cuda.synchronize()
    dl.check_status()
    _check(dl, b, cfg, rows=list(range(b.layout.T)))


def test_exact_kl_mid_vocab():
    b = synth.make_batch("mid", seed=3, with_ref=True)
    cfg = dart.Config(kl_mode=dart.KL_EXACT)
    dl = _run(b, cfg)
    rng = np.random.default_rng(2)
    _check(dl, b, cfg, rows=sorted(rng.choice(b.layout.T, 12, replace=False).tolist()))


def test_exact_kl_zero_for_identical_reference():
    b = synth.make_batch("small_multi", seed=10, with_ref=True)
    b.ref_logits = b.logits.clone()
    dl = _run(b, dart.Config(kl_mode=dart.KL_EXACT, beta_kl=0.5))
    assert float(dl.stats_dict()["sum_kl"]) <= 1e-5 * b.layout.T


def test_exact_kl_single_config_full_size_sampled():
    """BASELINE.json single config at full size (T = 61440, V = 152064 bf16,
    reference logits of the same shape) as `bench.py --kl exact` runs it:
    selection from the GPU's own step entropies, 10 sampled rows against the
    oracle row by row (kl_exact_row / token_row / token_loss composed as in
    `loss_pass`: l = surrogate + beta KL, dz = c invT [dl/dlogp (onehot - p)
    + beta p (log p - log q - KL)]), masked rows zero."""
    b = synth.make_batch("single", seed=0, device="cuda", with_ref=True)
    cfg = dart.Config(kl_mode=dart.KL_EXACT)
    cfgf = cfg.as_f32()
    dl = _run(b, cfg)
    L = b.layout
    keep = dl.keep.cpu().numpy()[:L.S]
    keep_same, _ = oracle_select_on(dl, b, cfgf)
    assert np.array_equal(keep, keep_same)
    nd = dl.norm_dict()
    tok_keep = np.repeat(keep, np.diff(L.step_tok_off)).astype(bool)
    A, _ = O.advantages(L.traj_reward, L.traj_group, L.traj_step_off, L.G)
    s_of_t = O.step_of_token(L.step_tok_off, L.T)
    tr_of_s = O.traj_of_step(L.traj_step_off, L.S)
    cfg0 = {**cfgf, "beta_kl": 0.0}
    beta, invT = cfgf["beta_kl"], cfgf["inv_temperature"]
    rng = np.random.default_rng(11)
    for t in sorted(rng.choice(np.nonzero(tok_keep)[0], 10, replace=False).tolist()):
        z = b.logits[t].float().cpu().numpy()
        zr = b.ref_logits[t].float().cpu().numpy()
        y = int(b.target[t])
        lse, logp, H, p = O.token_row(z, y, invT)
        klt, lpq = O.kl_exact_row(z, zr, invT)
        pg, dpg, w, r, clipped, _ = O.token_loss(logp, float(b.logp_old[t]), float(b.logp_rollout[t]),
                                                 float(b.logp_ref[t]), A[tr_of_s[s_of_t[t]]], cfg0)
        assert abs(float(dl.H[t]) - H) <= RTOL_ENT * H + ATOL_ENT
        assert abs(float(dl.logp[t]) - logp) <= ATOL_LOGP
        if min(abs(r - (1 - cfgf["eps_low"])), abs(r - (1 + cfgf["eps_high"]))) < 1e-5 * r:
            continue
        ell = pg + beta * klt
        assert abs(float(dl.ell[t]) - ell) <= RTOL_TOK * abs(ell) + ATOL_TOK
        c = nd["inv_norm"]
        onehot = np.zeros_like(p)
        onehot[y] = 1.0
        term = np.where(p > 0, p * (np.nan_to_num(lpq, nan=0.0, posinf=0.0, neginf=0.0) - klt), 0.0)
        dref = c * dpg * invT * (onehot - p) + c * beta * invT * term
        a = abs(c * invT)
        tol = bf16_ulp(dref) + a * (RTOL_TOK * abs(dpg) + ATOL_TOK) * np.abs(onehot - p)
        tol = tol + a * 4e-6 * p * (abs(dpg) + beta * (np.abs(lpq) + klt + 1.0))
        tol = tol + a * beta * p * 2e-5 * (1.0 + np.abs(lpq)) + 1e-38
        dz = dl.dlogits[t].float().cpu().numpy()
        err = np.abs(dz - dref)
        assert np.all(err <= tol), (t, np.argmax(err - tol), err.max())
    masked = torch.as_tensor(np.nonzero(~tok_keep)[0][:128], device="cuda")
    assert torch.all(dl.dlogits[masked] == 0)
    st = dl.stats_dict()
    ell_all = dl.ell.cpu().numpy().astype(np.float64)
    L_chk = np.sum(ell_all[tok_keep]) * nd["inv_norm"]
    assert abs(st["loss"] - L_chk) <= 1e-9 * np.sum(np.abs(ell_all[tok_keep])) * nd["inv_norm"] + 1e-15
