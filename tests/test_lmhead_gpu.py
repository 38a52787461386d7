"""GPU parity of the LM-head-fused forward (dart_lmhead_fwd)
against the float64 oracle: z = h W^T (oracle.lmhead_logits) followed by the
oracle's loss pass.

Two input families (synth.make_lmhead):
  * exact: integer h and W in 1/64 steps -- the tensor-core fp32 logits are
    exact, so the bar is the logits sweep's own: any tile,
    swizzle, descriptor or masking error shows up as a hard failure;
  * realistic: Gaussian operands; the fp32 accumulation error of the GEMM
    enters every output.  Its per-row bound E_t (DESIGN.md §9 "LM head")
    widens the tolerances by the first-order sensitivity of each output.
"""
import numpy as np
import pytest
import torch

from oracle import dart_oracle as O
from paper_2509_23866_b200 import dart, synth
from tests.gpu_helpers import ATOL_ENT, ATOL_LOGP, ATOL_TOK, RTOL_ENT, RTOL_TOK, oracle_select_on

pytestmark = pytest.mark.gpu

U32 = 2.0 ** -24          # fp32 unit roundoff


def run_lm(lb, cfg, runs=1):
    dev = torch.device("cuda")
    b = lb.batch
    dl = dart.DartLoss(b.layout, dart.whole_shard(b.layout), b.V, cfg, dev, with_grad=False)
    args = (lb.hidden.to(dev), lb.weight.to(dev), b.target.to(dev), b.logp_old.to(dev), b.logp_rollout.to(dev),
            b.logp_ref.to(dev))
    outs = []
    for _ in range(runs):
        dl.status.zero_()
        dl.forward_lmhead(*args)
        dl.select()
        torch.cuda.synchronize()
        outs.append([t.clone() for t in (dl.lse, dl.logp, dl.H, dl.ell, dl.dell, dl.step_H, dl.keep)])
    dl.check_status()
    return dl, outs


def gemm_bound(h, W, invT, exact):
    """Per-row bound on |z_gpu - z| * invT (0 for the exact family): bf16
    products are exact in fp32; each tcgen05.mma adds a K=16 slice to the fp32
    accumulator, so z is a sequential sum of ceil(d/16) slices and the classic
    bound gamma_n <= n u with n = d/16 + 4 (slack for the slice sums) applies
    to sum_k |h_tk W_vk|."""
    if exact:
        return np.zeros(h.shape[0])
    A = np.abs(h) @ np.abs(W).T
    n = -(-h.shape[1] // 16) + 4
    return n * U32 * A.max(axis=1) * invT


def compare_lm(dl, lb, cfg, exact):
    cfgf = cfg.as_f32()
    b = lb.batch
    L = b.layout
    h = lb.hidden.float().cpu().numpy()
    W = lb.weight.float().cpu().numpy()
    ob = b.oracle_dict(logits=False)
    ob["logits"] = O.lmhead_logits(h, W)
    invT = cfgf["inv_temperature"]
    E = gemm_bound(h, W, invT, exact)

    keep_gpu = dl.keep.cpu().numpy()[:L.S]
    keep_same, _ = oracle_select_on(dl, b, cfgf)
    assert np.array_equal(keep_gpu, keep_same), "selection differs from the oracle rule on the same values"
    ref = O.loss_pass(ob, cfgf, keep_override=keep_gpu, want_grad=False)

    lse, logp, H = dl.lse.cpu().numpy(), dl.logp.cpu().numpy(), dl.H.cpu().numpy()
    ell, dell = dl.ell.cpu().numpy(), dl.dell.cpu().numpy()
    err = dict(lse=np.abs(lse - ref["lse"]), logp=np.abs(logp - ref["logp"]), H=np.abs(H - ref["H"]))
    # first-order sensitivities: d lse = E, d logp <= 2E, d H <= E sum_v p_v |log p_v + H| <= 2 E (H + 1)
    tol_lse = RTOL_ENT * np.abs(ref["lse"]) + ATOL_ENT + E
    tol_logp = ATOL_LOGP + 2 * E
    tol_H = RTOL_ENT * np.abs(ref["H"]) + ATOL_ENT + 2 * E * (ref["H"] + 1.0)
    assert np.all(err["lse"] <= tol_lse), ("lse", err["lse"].max(), np.argmax(err["lse"] - tol_lse))
    assert np.all(err["logp"] <= tol_logp), ("logp", err["logp"].max())
    assert np.all(err["H"] <= tol_H), ("H", err["H"].max())
    r = ref["r"]
    near = (np.abs(r - (1 - cfgf["eps_low"])) < (1e-5 + 3 * E) * r) | \
        (np.abs(r - (1 + cfgf["eps_high"])) < (1e-5 + 3 * E) * r)
    ok = ~near
    dlogp = tol_logp
    ekl = cfgf["beta_kl"] * np.exp(ob["logp_ref"] - ref["logp"])
    tol_ell = RTOL_TOK * np.abs(ref["ell"]) + ATOL_TOK + 1.1 * np.abs(ref["dell"]) * (dlogp - ATOL_LOGP)
    tol_dell = RTOL_TOK * np.abs(ref["dell"]) + ATOL_TOK + 1.1 * (np.abs(ref["dell"]) + ekl) * (dlogp - ATOL_LOGP)
    assert np.all(np.abs(ell - ref["ell"])[ok] <= tol_ell[ok]), "ell"
    assert np.all(np.abs(dell - ref["dell"])[ok] <= tol_dell[ok]), "dell"
    sH = dl.step_H.cpu().numpy()[:L.S]
    n = np.diff(L.step_tok_off)
    tol_sH = RTOL_ENT * np.abs(ref["step_H"]) + ATOL_ENT + np.add.reduceat(tol_H - RTOL_ENT * np.abs(ref["H"]),
                                                                           L.step_tok_off[:-1]) / n
    assert np.all(np.abs(sH - ref["step_H"]) <= tol_sH), "step entropy"
    return {k: float(v.max()) for k, v in err.items()}, float(E.max())


@pytest.mark.parametrize("d,V,invT", [(256, 3000, 1.0), (200, 3000, 1.0), (64, 513, 1.0 / 0.7), (512, 5000, 1.0)])
def test_lmhead_exact_operands(d, V, invT):
    """Exact fp32 logits: ragged rows (T = 960 = 7.5 row blocks), vocabulary
    tail inside a tile and whole masked 32-column groups (V = 3000, 513),
    several vocabulary chunks (V = 5000: 20 tiles -> 3 chunks), a K tail
    (d = 200: the last 64-wide K block is 8 wide, zero-filled by TMA), a
    temperature."""
    lb = synth.make_lmhead("grid4x4x3x20@%d" % V, d, seed=3, exact=True, inv_temperature=invT)
    cfg = dart.Config(inv_temperature=invT, entropy_q=0.3)
    dl, _ = run_lm(lb, cfg)
    compare_lm(dl, lb, cfg, exact=True)


@pytest.mark.parametrize("d,V", [(512, 5000), (1024, 2304)])
def test_lmhead_realistic_operands(d, V):
    lb = synth.make_lmhead("grid3x4x3x24@%d" % V, d, seed=5)
    cfg = dart.Config()
    dl, _ = run_lm(lb, cfg)
    errs, emax = compare_lm(dl, lb, cfg, exact=False)
    print("max errors", errs, "E max", emax)


def test_lmhead_deterministic():
    lb = synth.make_lmhead("grid4x4x3x20@3000", 256, seed=7)
    _, outs = run_lm(lb, dart.Config(), runs=2)
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)


def test_lmhead_full_width_sampled_rows():
    """The bench's operand widths (d = 3584, V = 152064, Qwen2.5-7B head) on
    3 row blocks + a ragged tail; the oracle recomputes sampled rows' logits in
    float64 and checks lse / log-prob / entropy row by row."""
    layout = synth.config_layout("grid2x4x3x14@152064")[0]          # T = 336 rows
    lb = synth.make_lmhead(None, 3584, seed=9, layout=layout, V=synth.V_QWEN, device="cuda")
    cfg = dart.Config()
    dl, _ = run_lm(lb, cfg)
    invT = cfg.as_f32()["inv_temperature"]
    rows = np.array([0, 1, 127, 128, 200, 255, 256, 300, 335])
    h = lb.hidden[rows].float().cpu().numpy()
    W = lb.weight.float().cpu().numpy()
    z = O.lmhead_logits(h, W)
    E = gemm_bound(h, W, invT, exact=False)
    y = lb.batch.target.cpu().numpy()[rows]
    lse, logp, H = dl.lse.cpu().numpy()[rows], dl.logp.cpu().numpy()[rows], dl.H.cpu().numpy()[rows]
    for i in range(len(rows)):
        l_ref, lp_ref, H_ref, _ = O.token_row(z[i], int(y[i]), invT)
        assert abs(lse[i] - l_ref) <= RTOL_ENT * abs(l_ref) + ATOL_ENT + E[i], (rows[i], lse[i], l_ref)
        assert abs(logp[i] - lp_ref) <= ATOL_LOGP + 2 * E[i], (rows[i], logp[i], lp_ref)
        assert abs(H[i] - H_ref) <= RTOL_ENT * H_ref + ATOL_ENT + 2 * E[i] * (H_ref + 1), (rows[i], H[i], H_ref)


def test_lmhead_rejects_bad_operands():
    lb = synth.make_lmhead("grid2x2x2x8@300", 64, seed=1, exact=True)
    b = lb.batch
    dl = dart.DartLoss(b.layout, dart.whole_shard(b.layout), b.V, dart.Config(), "cuda", with_grad=False)
    with pytest.raises(dart.DartError):
        dl.forward_lmhead(lb.hidden.cuda().float(), lb.weight.cuda(), b.target.cuda(), b.logp_old.cuda(),
                          b.logp_rollout.cuda(), b.logp_ref.cuda())
    with pytest.raises(dart.DartError):       # d = 60: rows not 16-byte multiples
        dl.forward_lmhead(lb.hidden.cuda()[:, :60], lb.weight.cuda()[:, :60], b.target.cuda(), b.logp_old.cuda(),
                          b.logp_rollout.cuda(), b.logp_ref.cuda())


def test_lmhead_loss_only_backward_matches_oracle_loss():
    """dart_lmhead_fwd -> select -> dart_loss_bwd(dlogits = NULL): the loss and
    statistics of the pass without any [T, V] tensor (exact operands)."""
    lb = synth.make_lmhead("grid4x4x3x20@3000", 256, seed=11, exact=True)
    cfg = dart.Config(entropy_q=0.3)
    dl, _ = run_lm(lb, cfg)
    dl.backward()
    torch.cuda.synchronize()
    dl.check_status()
    cfgf = cfg.as_f32()
    ob = lb.batch.oracle_dict(logits=False)
    ob["logits"] = O.lmhead_logits(lb.hidden.float().numpy(), lb.weight.float().numpy())
    keep = dl.keep.cpu().numpy()[:lb.batch.layout.S]
    ref = O.loss_pass(ob, cfgf, keep_override=keep, want_grad=False)
    st = dl.stats_dict()
    scale = float(np.sum(np.abs(ref["c_tok"] * ref["ell"]))) + 1e-300
    assert abs(st["loss"] - ref["loss"]) <= RTOL_ENT * scale + 1e-12, (st["loss"], ref["loss"])
    for k in ("n_tok", "n_kept_tok", "n_kept_step"):
        assert st[k] == ref["stats"][k], k
    for k in ("sum_w", "sum_adv", "sum_H", "sum_kl"):
        assert abs(st[k] - ref["stats"][k]) <= 1e-5 * (abs(ref["stats"][k]) + 1.0), k


def test_lmhead_sharded_equals_unsharded():
    """Trajectory shards (virtual ranks, all-gather emulated by concatenation):
    each row's (m, s, u) is folded by one thread in tile order and chunk order,
    so every per-token value is bitwise the unsharded one."""
    from paper_2509_23866_b200 import dist as D
    lb = synth.make_lmhead("grid4x4x3x20@3000", 256, seed=13)
    b = lb.batch
    cfg = dart.Config()
    ref, _ = run_lm(lb, cfg)
    shards = D.shard_layout(b.layout, 3)
    dls = []
    for sh in shards:
        dl = dart.DartLoss(b.layout, sh, b.V, cfg, "cuda", group=False, world_shards=shards, with_grad=False)
        sl = slice(sh.tok_begin, sh.tok_end)
        dl.forward_lmhead(lb.hidden[sl].cuda().contiguous(), lb.weight.cuda(), b.target[sl].cuda().contiguous(),
                          b.logp_old[sl].cuda().contiguous(), b.logp_rollout[sl].cuda().contiguous(),
                          b.logp_ref[sl].cuda().contiguous())
        dls.append(dl)
    S_pad = dls[0].S_pad
    gathered = torch.zeros(len(shards) * S_pad, dtype=torch.float32, device="cuda")
    for r, (dl, sh) in enumerate(zip(dls, shards)):
        gathered[r * S_pad: r * S_pad + sh.S_loc] = dl.step_H[:sh.S_loc]
    for dl in dls:
        dl.set_gathered(gathered)
        dl.select()
    torch.cuda.synchronize()
    for dl, sh in zip(dls, shards):
        dl.check_status()
        sl = slice(sh.tok_begin, sh.tok_end)
        assert torch.equal(dl.keep[:b.layout.S], ref.keep[:b.layout.S])
        for a, c in ((dl.lse, ref.lse[sl]), (dl.logp, ref.logp[sl]), (dl.H, ref.H[sl]), (dl.ell, ref.ell[sl])):
            assert torch.equal(a, c)


def test_lmhead_full_vocab_exact_operands():
    """V = 152064 (594 tiles, 75 vocabulary chunks, last chunk 2 tiles) with
    exact operands and a small d: every output against the oracle at the
    logits sweep's tolerances."""
    layout = synth.config_layout("grid1x2x2x40@152064")[0]          # T = 160 rows (2 blocks, ragged)
    lb = synth.make_lmhead(None, 64, seed=17, layout=layout, V=synth.V_QWEN, exact=True)
    cfg = dart.Config(entropy_q=0.3)
    dl, _ = run_lm(lb, cfg)
    compare_lm(dl, lb, cfg, exact=True)
