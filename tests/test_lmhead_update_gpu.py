"""GPU parity of the LM-head backward (training half):
dart_lmhead_bwd -- the kept rows gathered, z = h W^T recomputed on the
tensor cores and turned into bf16 dz = dL/dz in the TMEM epilogue -- and the
update pass around it (paper_2509_23866_b200.lmhead.LmHeadUpdate: forward at
theta, dart_lmhead_bwd, dh = dz W and dW = dz^T h_kept on cuBLAS), against
the oracle: float64 z = h W^T (oracle.lmhead_logits) -> the loss pass ->
dz -> oracle.lmhead_grads.

Error model.  The GPU's fp32 logits carry the GEMM error
E_t = (ceil(d/16) + 4) u max_v sum_k |h_tk W_vk| (0 for the exact-operand
family), so p_v carries (P_REL + 2 E invT) p_v and g_t = c dell_t invT the
per-token tolerance of dell widened by 4 E invT:
  |dz - dz_ref| <= ulp_bf16(dz_ref) + dg |delta - p| + (|g| + dg)(P_REL + 2 E invT) max(p, onehot).
dh / dW add the library GEMM's fp32 accumulation error, bounded for any
summation order by n u per unit of sum |dz| |W| (resp. |dz| |h|)."""
import numpy as np
import pytest
import torch

from oracle import dart_oracle as O
from paper_2509_23866_b200 import dart, lmhead, synth
from tests.gpu_helpers import ATOL_LOGP, ATOL_TOK, P_REL, RTOL_ENT, RTOL_TOK, bf16_ulp

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


def run_update(lb, cfg, keep, norm, chunk_rows=None):
    b = lb.batch
    up = lmhead.LmHeadUpdate(b.layout, b.V, lb.hidden.shape[1], cfg, "cuda", chunk_rows=chunk_rows)
    dh, dW = up.run(lb.hidden.cuda(), lb.weight.cuda(), b.target.cuda(), b.logp_old.cuda(), b.logp_rollout.cuda(),
                    b.logp_ref.cuda(), keep, norm)
    torch.cuda.synchronize()
    up.check_status()
    return up, dh, dW


def gemm_E(h, W, d, exact):
    return 0.0 if exact else float((-(-d // 16) + 4) * U * (np.abs(h) @ np.abs(W).T).max())


def dz_tol(dref, p, y, g, dg, Ez, invT):
    onehot = np.zeros_like(p)
    onehot[y] = 1.0
    return bf16_ulp(dref) + dg * np.abs(onehot - p) + (abs(g) + dg) * (P_REL + 2 * Ez * invT) * np.maximum(p, onehot) \
        + abs(g) * 2.0 ** -125 + 1e-38


def near_clip(r, cfgf, win):
    return min(abs(r - (1 - cfgf["eps_low"])), abs(r - (1 + cfgf["eps_high"]))) < win * r


@pytest.mark.parametrize("d,V,chunk_rows,exact", [(256, 3000, None, False), (512, 5000, 500, False),
                                                 (128, 2048, 150, True), (64, 776, None, True)])
def test_lmhead_update_matches_oracle(d, V, chunk_rows, exact):
    lb = synth.make_lmhead("grid3x4x3x24@%d" % V, d, seed=21, exact=exact)
    # wide clip bounds: no ratio sits near a clip boundary, so no token's surrogate
    # branch can flip under the logits' GEMM error and dW (a sum over all rows) is
    # comparable element by element; the paper's bounds are covered row-wise below
    cfg = dart.Config(entropy_q=0.3, eps_low=0.95, eps_high=0.95)
    check_update(lb, cfg, chunk_rows, exact, expect_chunks=bool(chunk_rows))


def check_update(lb, cfg, chunk_rows, exact, expect_chunks=False):
    """The update pass on `lb` against the oracle (the error model above)."""
    d, V = lb.hidden.shape[1], lb.batch.V
    old = old_pass(lb, cfg)
    up, dh, dW = run_update(lb, cfg, old.keep, old.norm, chunk_rows)
    if expect_chunks:              # (chunks are whole trajectories: a fuzz batch may have one)
        assert len(up.chunks) > 1
    cfgf = cfg.as_f32()
    invT = cfgf["inv_temperature"]
    L = lb.batch.layout
    h = lb.hidden.float().numpy()
    W = lb.weight.float().numpy()
    ob = lb.batch.oracle_dict(logits=False)
    ob["logits"] = O.lmhead_logits(h, W)
    keep = old.keep.cpu().numpy()[:L.S]
    ref = O.loss_pass(ob, cfgf, keep_override=keep)
    T = L.T
    Ez = gemm_E(h, W, d, exact)
    # --- the gathered rows: exactly the rows of kept steps, in order; their hidden states bitwise
    tok_keep = np.repeat(keep, np.diff(L.step_tok_off)).astype(bool)
    K = int(tok_keep.sum())
    assert up.last_n_kept == K
    if not chunk_rows:
        assert np.array_equal(up.kept_rows[:K].cpu().numpy(), np.nonzero(tok_keep)[0])
        assert torch.equal(up.h_kept[:K].cpu(), lb.hidden[np.nonzero(tok_keep)[0]])
        # --- dz of every kept row against the oracle, element by element
        dz_gpu = up.dz[:K].float().cpu().numpy()
        for i, t in enumerate(np.nonzero(tok_keep)[0]):
            g = ref["c_tok"][t] * ref["dell"][t] * invT
            _, p = O.log_softmax_row(ob["logits"][t], invT)
            dg = abs(ref["c_tok"][t] * invT) * ((RTOL_TOK + 4 * Ez) * abs(ref["dell"][t]) + ATOL_TOK)
            tol = dz_tol(ref["dz"][t], p, int(ob["target"][t]), g, dg, Ez, invT)
            err = np.abs(dz_gpu[i] - ref["dz"][t])
            assert np.all(err <= tol), (t, err.max(), np.argmax(err - tol))
    # --- dh, dW through the library GEMMs
    dz = np.stack([ref["dz"][t] for t in range(T)])
    dh_ref, dW_ref = O.lmhead_grads(dz, h, W)
    rel = (2.0 ** -8 + (RTOL_TOK + 4 * Ez) + 2 * Ez * invT + ATOL_TOK / np.maximum(np.abs(ref["dell"]), 1e-30))[:, None]
    a = np.zeros_like(dz)
    beta = cfgf["beta_kl"]
    for t in np.nonzero(ref["c_tok"])[0]:
        p_t = O.log_softmax_row(ob["logits"][t], invT)[1]
        a[t] = abs(ref["c_tok"][t] * ref["dell"][t]) * invT * (P_REL + 2 * Ez * invT) * p_t
        # dell's sensitivity to the log-prob error: |d dell / d logp| = |-w A r act + beta e^d|
        # times ATOL_LOGP + 4 Ez invT (the forward's lse and the dz kernel's recomputed z are two
        # GEMMs, each within Ez) -- an absolute term that matters where dell itself is ~0
        # (A = 0 and logp_ref = logp: the fuzz's degenerate rows, tests/test_fuzz_paths_gpu.py)
        sens = abs(ref["w"][t] * ref["A_tok"][t] * ref["r"][t]) + beta * np.exp(ob["logp_ref"][t] - ref["logp"][t])
        onehot = np.zeros_like(p_t)
        onehot[int(ob["target"][t])] = 1.0
        # ... times |delta - p| as the GPU sees it: p within (P_REL + 4 Ez invT) p (near-one-hot rows)
        a[t] += abs(ref["c_tok"][t]) * invT * sens * (ATOL_LOGP + 4 * Ez * invT) * \
            (np.abs(onehot - p_t) + (P_REL + 4 * Ez * invT) * p_t)
    tol_dh = (rel + V * U) * (np.abs(dz) @ np.abs(W)) + a @ np.abs(W) + 1e-30
    tol_dW = ((rel + T * U) * np.abs(dz) + a).T @ np.abs(h) + 1e-30
    e_dh = np.abs(dh.cpu().numpy() - dh_ref)
    e_dW = np.abs(dW.cpu().numpy() - dW_ref)
    bad = np.argwhere(e_dh > tol_dh)
    assert bad.size == 0, ("dh", bad[:5], e_dh[tuple(bad[0])], tol_dh[tuple(bad[0])])
    assert np.all(e_dW <= tol_dW), ("dW", e_dW.max())
    assert np.all(dh.cpu().numpy()[~tok_keep] == 0)          # rows of masked steps: no gradient
    st = up.stats_dict()
    scale = float(np.sum(np.abs(ref["c_tok"] * ref["ell"]))) + 1e-300
    assert abs(st["loss"] - ref["loss"]) <= (RTOL_ENT + 4 * Ez) * scale + 1e-12, (st["loss"], ref["loss"])
    assert st["n_kept_tok"] == ref["stats"]["n_kept_tok"] == K


def test_lmhead_update_chunking_invariance():
    """Chunks are virtual ranks: every dz row and hence every dh row is the
    same whatever the chunking (dz bitwise; dh up to the library GEMM's
    shape-dependent kernel choice); dW only through the chunk sum order."""
    lb = synth.make_lmhead("grid3x4x3x24@3000", 256, seed=23)
    cfg = dart.Config()
    old = old_pass(lb, cfg)
    up1, dh1, dW1 = run_update(lb, cfg, old.keep, old.norm, None)
    K = up1.last_n_kept
    dz1 = up1.dz[:K].clone()
    up2, dh2, dW2 = run_update(lb, cfg, old.keep, old.norm, 150)
    assert len(up2.chunks) > 2
    loss1, loss2 = up1.stats_dict()["loss"], up2.stats_dict()["loss"]
    assert abs(loss1 - loss2) <= 1e-12 * abs(loss1) + 1e-15
    # reassemble the chunked run's dz rows: rerun chunk by chunk and compare
    off = 0
    b = lb.batch
    for c, p in zip(up2.chunks, up2.parts):
        r0, r1 = c.tok_begin, c.tok_end
        sl = slice(r0, r1)
        p.forward_lmhead(lb.hidden[sl].cuda(), lb.weight.cuda(), b.target[sl].cuda(), b.logp_old[sl].cuda(),
                         b.logp_rollout[sl].cuda(), b.logp_ref[sl].cuda())
        p.backward_lmhead(up2.dz, up2.h_kept, up2.kept_rows, up2.n_kept, keep=old.keep, norm=old.norm)
        k = int(up2.n_kept.item())
        assert torch.equal(up2.dz[:k], dz1[off:off + k])
        off += k
    assert off == K
    assert torch.allclose(dh1, dh2, rtol=1e-5, atol=1e-9)
    assert torch.allclose(dW1, dW2, rtol=1e-4, atol=1e-7)


def test_theta_old_one_object_equals_update_pass():
    """theta = theta_old: forward_lmhead -> select -> backward_lmhead on ONE
    DartLoss gives bitwise the dz rows of the update pass run with that
    object's own mask."""
    lb = synth.make_lmhead("grid3x4x3x24@3000", 256, seed=29)
    b = lb.batch
    cfg = dart.Config()
    dl = old_pass(lb, cfg)
    T = b.layout.T
    dz = torch.empty((T, b.V), dtype=torch.bfloat16, device="cuda")
    hk = torch.empty((T, 256), dtype=torch.bfloat16, device="cuda")
    kr = torch.empty(T, dtype=torch.int32, device="cuda")
    nk = torch.zeros(1, dtype=torch.int64, device="cuda")
    dl.backward_lmhead(dz, hk, kr, nk)
    torch.cuda.synchronize()
    up, _, _ = run_update(lb, cfg, dl.keep, dl.norm)
    K = int(nk.item())
    assert K == up.last_n_kept > 0
    assert torch.equal(dz[:K], up.dz[:K]) and torch.equal(kr[:K], up.kept_rows[:K])
    assert dl.stats_dict()["loss"] == up.stats_dict()["loss"]


def test_lmhead_update_default_clip_rows():
    """Paper clip bounds (0.2 / 0.28): dz row by row, skipping rows whose ratio
    sits within the GEMM / fp32 error of a clip boundary."""
    lb = synth.make_lmhead("grid3x4x3x24@3000", 256, seed=25)
    cfg = dart.Config()
    old = old_pass(lb, cfg)
    up, dh, _ = run_update(lb, cfg, old.keep, old.norm)
    cfgf = cfg.as_f32()
    L = lb.batch.layout
    h, W = lb.hidden.float().numpy(), lb.weight.float().numpy()
    ob = lb.batch.oracle_dict(logits=False)
    ob["logits"] = O.lmhead_logits(h, W)
    keep = old.keep.cpu().numpy()[:L.S]
    ref = O.loss_pass(ob, cfgf, keep_override=keep)
    Ez = gemm_E(h, W, 256, False)
    rows = np.nonzero(np.repeat(keep, np.diff(L.step_tok_off)).astype(bool))[0]
    dz_gpu = up.dz[:len(rows)].float().cpu().numpy()
    checked = 0
    for i, t in enumerate(rows):
        if near_clip(ref["r"][t], cfgf, 1e-5 + 4 * Ez):
            continue
        g = ref["c_tok"][t] * ref["dell"][t]
        _, p = O.log_softmax_row(ob["logits"][t])
        dg = abs(ref["c_tok"][t]) * ((RTOL_TOK + 4 * Ez) * abs(ref["dell"][t]) + ATOL_TOK)
        tol = dz_tol(ref["dz"][t], p, int(ob["target"][t]), g, dg, Ez, 1.0)
        assert np.all(np.abs(dz_gpu[i] - ref["dz"][t]) <= tol), t
        checked += 1
    assert checked > 0.9 * len(rows)


def test_lmhead_update_full_size_sampled_rows():
    """`bench.py --lmhead --update` at full size (T = 61440, d = 3584,
    V = 152064): dz and dh on sampled kept rows against the oracle (z_t = h_t
    W^T in float64 -> the loss terms -> dz_t -> dz_t W), masked rows' dh
    exactly zero, the gathered rows exactly the kept steps' rows."""
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
    up, dh, dW = run_update(lb, cfg, old.keep, old.norm)
    tok_keep = np.repeat(keep, np.diff(L.step_tok_off)).astype(bool)
    rows_k = np.nonzero(tok_keep)[0]
    assert up.last_n_kept == len(rows_k)
    assert np.array_equal(up.kept_rows[:len(rows_k)].cpu().numpy(), rows_k)
    inv_norm = 1.0 / float(tok_keep.sum())                    # TOKEN_MEAN_KEPT
    A, _ = O.advantages(L.traj_reward, L.traj_group, L.traj_step_off, L.G)
    s_of_t = O.step_of_token(L.step_tok_off, L.T)
    tr_of_s = O.traj_of_step(L.traj_step_off, L.S)
    W = lb.weight.float().cpu().numpy().astype(np.float64)
    rng = np.random.default_rng(5)
    pick = sorted(rng.choice(len(rows_k), 6, replace=False).tolist())
    dh_np = dh.cpu().numpy()
    for i in pick:
        t = int(rows_k[i])
        h_t = lb.hidden[t].float().cpu().numpy().astype(np.float64)
        z = O.lmhead_logits(h_t[None, :], W)[0]
        y = int(b.target[t])
        lse, logp, H, p = O.token_row(z, y)
        ell, dell, w, r, clipped, kl = O.token_loss(logp, float(b.logp_old[t]), float(b.logp_rollout[t]),
                                                    float(b.logp_ref[t]), A[tr_of_s[s_of_t[t]]], cfgf)
        Ez = float((-(-d // 16) + 4) * U * (np.abs(h_t) @ np.abs(W).T).max())
        if near_clip(r, cfgf, 1e-5 + 4 * Ez):
            continue
        g = inv_norm * dell
        onehot = np.zeros_like(p)
        onehot[y] = 1.0
        dref = g * (onehot - p)
        dg = inv_norm * ((RTOL_TOK + 4 * Ez) * abs(dell) + ATOL_TOK)
        tol = dz_tol(dref, p, y, g, dg, Ez, 1.0)
        dz_row = up.dz[i].float().cpu().numpy()
        assert np.all(np.abs(dz_row - dref) <= tol), (t, np.abs(dz_row - dref).max())
        dh_ref = dref @ W
        rel = 2.0 ** -8 + RTOL_TOK + 6 * Ez + ATOL_TOK / max(abs(dell), 1e-30)
        a = abs(g) * (P_REL + 2 * Ez) * p
        tol_h = (rel + V * U) * (np.abs(dref) @ np.abs(W)) + a @ np.abs(W) + 1e-30
        err = np.abs(dh_np[t] - dh_ref)
        assert np.all(err <= tol_h), (t, err.max())
    masked = np.nonzero(~tok_keep)[0][:256]
    assert np.all(dh_np[masked] == 0)
    assert np.all(np.isfinite(dW[:4096].cpu().numpy()))
    st = up.stats_dict()
    assert st["n_kept_tok"] == tok_keep.sum()
