"""GPU parity of the LM-head update pass (training half;
paper_2509_23866_b200.lmhead.LmHeadUpdate): per chunk z = h W^T (tcgen05),
the fused loss kernel (dz in bf16), dh = dz W and dW += dz^T h (tcgen05),
against the oracle's dz pushed through oracle.lmhead_grads.

Error model: dz leaves the fused kernel rounded to bf16
(<= 2^-9 relative) after an fp32 computation whose row factor g = c dell / T
carries the per-token tolerance of dell (1e-5 relative + 2e-6 absolute, i.e.
2e-6 / |dell_t| relative to the row) and the logits' own GEMM error 2 E_t
from z = h W^T; the two GEMMs add fp32 accumulation error (ceil(K/16) + 4) u
per unit of sum |dz| |W| (resp. sum |dz| |h|).  Besides, each element of dz carries
the fp32 error of p_v itself, |g_t| (P_REL + 2 E) p_tv absolute (the gradient
sweep's error model, tests/gpu_helpers.grad_tol): for a peaked row the target
element g (1 - p_y) is pure cancellation.  So with
rel_t = 2^-8 + 2e-5 + 2e-6 / |dell_t| + 2 E and a_tv = |g_t| (P_REL + 2 E) p_tv:
|dh - dh_ref| <= (rel_t + n_V u) (|dz_ref| |W|) + a |W|  and
|dW - dW_ref| <= ((rel_t + n_T u) |dz_ref| + a)^T |h|  elementwise."""
import numpy as np
import pytest
import torch

from oracle import dart_oracle as O
from paper_2509_23866_b200 import dart, lmhead, synth
from tests.gpu_helpers import ATOL_TOK, P_REL, RTOL_ENT

pytestmark = pytest.mark.gpu

U = 2.0 ** -24


def old_pass(lb, cfg):
    b = lb.batch
    dl = dart.DartLoss(b.layout, dart.whole_shard(b.layout), b.V, cfg, "cuda", with_grad=False)
    dl.forward_lmhead(lb.hidden.cuda(), lb.weight.cuda(), b.target.cuda(), b.logp_old.cuda(), b.logp_rollout.cuda(),
                      b.logp_ref.cuda())
    dl.select()
    torch.cuda.synchronize()
    dl.check_status()
    return dl


def p_term(ob, ref, cfgf, Ez):
    """a_tv = |g_t| (P_REL + 2 E) p_tv, g_t = c_t dell_t invT (0 for masked rows)."""
    invT = cfgf["inv_temperature"]
    z = ob["logits"]
    a = np.zeros_like(z)
    g = np.abs(ref["c_tok"] * ref["dell"]) * invT
    for t in np.nonzero(g)[0]:
        a[t] = g[t] * (P_REL + 2 * Ez * invT) * O.log_softmax_row(z[t], invT)[1]
    return a


def run_update(lb, cfg, keep, norm, chunk_rows):
    b = lb.batch
    up = lmhead.LmHeadUpdate(b.layout, b.V, lb.hidden.shape[1], cfg, "cuda", chunk_rows=chunk_rows)
    dh, dW = up.run(lb.hidden.cuda(), lb.weight.cuda(), b.target.cuda(), b.logp_old.cuda(), b.logp_rollout.cuda(),
                    b.logp_ref.cuda(), keep, norm)
    torch.cuda.synchronize()
    up.check_status()
    return up, dh, dW


@pytest.mark.parametrize("d,V,chunk_rows,exact", [(256, 3000, 200, False), (512, 5000, 500, False),
                                                 (128, 2048, 150, True)])
def test_lmhead_update_matches_oracle(d, V, chunk_rows, exact):
    lb = synth.make_lmhead("grid3x4x3x24@%d" % V, d, seed=21, exact=exact)
    # wide clip bounds: no ratio sits near a clip boundary, so no token's
    # surrogate branch can flip under the logits' GEMM error and dW (a sum over
    # all rows) is comparable element by element; the clipped branches are
    # covered row-wise below and by the fused-kernel tests
    cfg = dart.Config(entropy_q=0.3, eps_low=0.95, eps_high=0.95)
    old = old_pass(lb, cfg)
    up, dh, dW = run_update(lb, cfg, old.keep, old.norm, chunk_rows)
    assert len(up.chunks) > 1
    cfgf = cfg.as_f32()
    L = lb.batch.layout
    h = lb.hidden.float().numpy()
    W = lb.weight.float().numpy()
    ob = lb.batch.oracle_dict(logits=False)
    ob["logits"] = O.lmhead_logits(h, W)
    keep = old.keep.cpu().numpy()[:L.S]
    ref = O.loss_pass(ob, cfgf, keep_override=keep)
    T = L.T
    dz = np.stack([ref["dz"][t] for t in range(T)])
    dh_ref, dW_ref = O.lmhead_grads(dz, h, W)
    # the logits' own fp32 GEMM error (0 for exact operands)
    Ez = 0.0 if exact else float(((-(-d // 16) + 4) * U * (np.abs(h) @ np.abs(W).T).max()))
    rel = (2.0 ** -8 + 2e-5 + 2 * Ez * cfgf["inv_temperature"]
           + ATOL_TOK / np.maximum(np.abs(ref["dell"]), 1e-30))[:, None]
    a = p_term(ob, ref, cfgf, Ez)
    tol_dh = (rel + (-(-V // 16) + 4) * U) * (np.abs(dz) @ np.abs(W)) + a @ np.abs(W) + 1e-30
    tol_dW = ((rel + (-(-T // 16) + 4) * U) * np.abs(dz) + a).T @ np.abs(h) + 1e-30
    e_dh = np.abs(dh.cpu().numpy() - dh_ref)
    e_dW = np.abs(dW.cpu().numpy() - dW_ref)
    bad = np.argwhere(e_dh > tol_dh)
    assert bad.size == 0, ("dh", bad[:5], e_dh[tuple(bad[0])], tol_dh[tuple(bad[0])], ref["dell"][bad[0][0]],
                           ref["r"][bad[0][0]], ref["c_tok"][bad[0][0]])
    assert np.all(e_dW <= tol_dW), ("dW", e_dW.max())
    # rows of masked steps carry no gradient at all
    tok_keep = np.repeat(keep, np.diff(L.step_tok_off)).astype(bool)
    assert np.all(dh.cpu().numpy()[~tok_keep] == 0)
    st = up.stats_dict()
    scale = float(np.sum(np.abs(ref["c_tok"] * ref["ell"]))) + 1e-300
    assert abs(st["loss"] - ref["loss"]) <= (RTOL_ENT + 4 * Ez) * scale + 1e-12, (st["loss"], ref["loss"])
    assert st["n_kept_tok"] == ref["stats"]["n_kept_tok"]


def test_lmhead_update_chunking_invariance():
    """dh rows do not depend on the chunking (each element is one GEMM row with
    a fixed K order); dW only through the fp32 accumulation order of chunks."""
    lb = synth.make_lmhead("grid3x4x3x24@3000", 256, seed=23)
    cfg = dart.Config()
    old = old_pass(lb, cfg)
    _, dh1, dW1 = run_update(lb, cfg, old.keep, old.norm, 150)
    _, dh2, dW2 = run_update(lb, cfg, old.keep, old.norm, 100000)
    assert torch.equal(dh1, dh2)
    assert torch.allclose(dW1, dW2, rtol=1e-5, atol=1e-7)


def test_lmhead_update_default_clip_rows():
    """Paper clip bounds (0.2 / 0.28): dh row by row, skipping rows whose ratio
    sits within the GEMM / fp32 error of a clip boundary."""
    lb = synth.make_lmhead("grid3x4x3x24@3000", 256, seed=25)
    cfg = dart.Config()
    old = old_pass(lb, cfg)
    _, dh, _ = run_update(lb, cfg, old.keep, old.norm, 200)
    cfgf = cfg.as_f32()
    L = lb.batch.layout
    h, W = lb.hidden.float().numpy(), lb.weight.float().numpy()
    ob = lb.batch.oracle_dict(logits=False)
    ob["logits"] = O.lmhead_logits(h, W)
    keep = old.keep.cpu().numpy()[:L.S]
    ref = O.loss_pass(ob, cfgf, keep_override=keep)
    dz = np.stack([ref["dz"][t] for t in range(L.T)])
    dh_ref, _ = O.lmhead_grads(dz, h, W)
    Ez = float(((-(-256 // 16) + 4) * U * (np.abs(h) @ np.abs(W).T).max()))
    r = ref["r"]
    win = 1e-5 + 4 * Ez
    near = (np.abs(r - (1 - cfgf["eps_low"])) < win * r) | (np.abs(r - (1 + cfgf["eps_high"])) < win * r)
    rel = (2.0 ** -8 + 2e-5 + 2 * Ez + ATOL_TOK / np.maximum(np.abs(ref["dell"]), 1e-30))[:, None]
    tol = (rel + (-(-3000 // 16) + 4) * U) * (np.abs(dz) @ np.abs(W)) + p_term(ob, ref, cfgf, Ez) @ np.abs(W) + 1e-30
    err = np.abs(dh.cpu().numpy() - dh_ref)
    bad = np.argwhere((err > tol) & ~near[:, None])
    assert bad.size == 0, (bad[:5], err[tuple(bad[0])], tol[tuple(bad[0])], ref["dell"][bad[0][0]], r[bad[0][0]])


def test_lmhead_update_full_size_sampled_rows():
    """`bench.py --lmhead --update` at full size (T = 61440, d = 3584,
    V = 152064, 8192-row chunks): dh on sampled rows against the oracle
    (z_t = h_t W^T in float64 -> the loss terms -> dz_t -> dz_t W, same error
    model as above), masked rows' dh exactly zero.  The mask is the old pass's
    (checked against the oracle's rule on the GPU's own step entropies, the
    same-precision decision); the normaliser is recomputed from it here."""
    layout, V, _, _ = synth.config_layout("single", seed=0)
    d = 3584
    lb = synth.make_lmhead(None, d, seed=0, device="cuda", layout=layout, V=V)
    b = lb.batch
    cfg = dart.Config()
    cfgf = cfg.as_f32()
    old = old_pass(lb, cfg)
    L = b.layout
    from tests.gpu_helpers import oracle_select_on
    keep_same, _ = oracle_select_on(old, b, cfgf)
    keep = old.keep.cpu().numpy()[:L.S]
    assert np.array_equal(keep, keep_same)
    up, dh, dW = run_update(lb, cfg, old.keep, old.norm, 8192)
    assert len(up.chunks) == 8
    tok_keep = np.repeat(keep, np.diff(L.step_tok_off)).astype(bool)
    inv_norm = 1.0 / float(tok_keep.sum())                    # TOKEN_MEAN_KEPT
    A, _ = O.advantages(L.traj_reward, L.traj_group, L.traj_step_off, L.G)
    s_of_t = O.step_of_token(L.step_tok_off, L.T)
    tr_of_s = O.traj_of_step(L.traj_step_off, L.S)
    W = lb.weight.float().cpu().numpy().astype(np.float64)
    rng = np.random.default_rng(5)
    rows = rng.choice(np.nonzero(tok_keep)[0], 4, replace=False).tolist()
    dh_np = dh.cpu().numpy()
    for t in rows:
        h_t = lb.hidden[t].float().cpu().numpy().astype(np.float64)
        z = O.lmhead_logits(h_t[None, :], W)[0]
        y = int(b.target[t])
        lse, logp, H, p = O.token_row(z, y)
        ell, dell, w, r, clipped, kl = O.token_loss(logp, float(b.logp_old[t]), float(b.logp_rollout[t]),
                                                    float(b.logp_ref[t]), A[tr_of_s[s_of_t[t]]], cfgf)
        Ez = float((-(-d // 16) + 4) * U * (np.abs(h_t) @ np.abs(W).T).max())
        if min(abs(r - (1 - cfgf["eps_low"])), abs(r - (1 + cfgf["eps_high"]))) < (1e-5 + 4 * Ez) * r:
            continue
        g = inv_norm * dell
        onehot = np.zeros_like(p)
        onehot[y] = 1.0
        dz = g * (onehot - p)
        dh_ref = dz @ W            # lmhead_grads' dL/dh row (its [V, d] dW product is not needed here)
        rel = 2.0 ** -8 + 2e-5 + 2 * Ez + ATOL_TOK / max(abs(dell), 1e-30)
        a = abs(g) * (P_REL + 2 * Ez) * p
        tol = (rel + (-(-V // 16) + 4) * U) * (np.abs(dz) @ np.abs(W)) + a @ np.abs(W) + 1e-30
        err = np.abs(dh_np[t] - dh_ref)
        assert np.all(err <= tol), (t, err.max(), tol[np.argmax(err - tol)])
    masked = np.nonzero(~tok_keep)[0][:256]
    assert np.all(dh_np[masked] == 0)
    assert np.all(np.isfinite(dW[:4096].cpu().numpy()))
    st = up.stats_dict()
    assert st["n_kept_tok"] == tok_keep.sum()


def test_lmhead_update_dw_group_invariance():
    """Grouping chunks into one dW GEMM (dw_group) changes only the fp32
    accumulation order of dW; dh is bitwise the same."""
    lb = synth.make_lmhead("grid3x4x3x24@3000", 256, seed=27)
    cfg = dart.Config()
    old = old_pass(lb, cfg)
    b = lb.batch
    outs = []
    for g in (1, 3):
        up = lmhead.LmHeadUpdate(b.layout, b.V, 256, cfg, "cuda", chunk_rows=150, dw_group=g)
        dh, dW = up.run(lb.hidden.cuda(), lb.weight.cuda(), b.target.cuda(), b.logp_old.cuda(),
                        b.logp_rollout.cuda(), b.logp_ref.cuda(), old.keep, old.norm)
        torch.cuda.synchronize()
        up.check_status()
        assert len(up.chunks) > 3
        outs.append((dh, dW))
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.allclose(outs[0][1], outs[1][1], rtol=1e-5, atol=1e-7)
