"""The chunk-streamed pass at a BASELINE.json config's full size, in the
launch configuration `bench.py --config long --stream-rows 32768 --pool 3`
times: 819,200 tokens (16 tasks x 8 rollouts x 50 steps x 128 tokens), 26
chunks through a pool of 3 logits buffers.  The oracle checks what it can
compute one by one -- advantages and group validity exactly, the selection
rule on the GPU's own step entropies (the same-precision decision), sampled
rows' lse / entropy / log-prob / loss terms and gradient rows -- and the
rest by properties (masked rows zero, loss = sum of the GPU's kept terms)."""
import numpy as np
import pytest
import torch

from oracle import dart_oracle as O
from paper_2509_23866_b200 import dart, synth
from paper_2509_23866_b200.stream import StreamedPass
from tests.gpu_helpers import ATOL_ENT, ATOL_LOGP, ATOL_TOK, RTOL_ENT, RTOL_TOK, grad_tol

pytestmark = pytest.mark.gpu


def test_long_config_streamed_full_size_sampled():
    dev = torch.device("cuda")
    layout, V, dtype, _ = synth.config_layout("long", seed=0)
    cfg = dart.Config()
    cfgf = cfg.as_f32()
    sp = StreamedPass(layout, V, cfg, dev, max_rows=32768, pool=3, logits_dtype=dtype)
    P, rows = sp.P, sp.rows
    assert len(sp.chunks) > P                        # chunks really cycle through the pool
    # pool contents: the config's value recipe on P x rows synthetic rows (as bench.run_streamed)
    nstep = -(-P * rows // 64)
    sub = synth.Layout(G=1, traj_group=np.zeros(1, np.int32), traj_reward=np.ones(1, np.float32),
                       traj_step_off=np.array([0, nstep], np.int64),
                       step_tok_off=np.minimum(np.arange(nstep + 1, dtype=np.int64) * 64, P * rows),
                       step_fork=np.random.default_rng(0).random(nstep) < 0.3)
    sb = synth.make_batch("long", seed=0, device=dev, layout=sub, V=V, dtype=dtype)
    for k in range(P):
        sp.pool_logits[k].copy_(sb.logits[k * rows:(k + 1) * rows])
    T = layout.T
    src = np.empty(T, dtype=np.int64)                # global token -> pool row (slot * rows + r)
    for i, c in enumerate(sp.chunks):
        src[c.tok_begin:c.tok_end] = (i % P) * rows + np.arange(c.T_loc)
    idx = torch.as_tensor(src, device=dev)
    target, lo, lr, lref = (x[idx].contiguous() for x in (sb.target, sb.logp_old, sb.logp_rollout, sb.logp_ref))

    rng = np.random.default_rng(3)
    sample = sorted(rng.choice(T, 14, replace=False).tolist())
    chunk_of = np.searchsorted([c.tok_end for c in sp.chunks], np.asarray(sample), side="right")
    got = {}

    def consume(i, dz):
        c = sp.chunks[i]
        for t in sample:
            if c.tok_begin <= t < c.tok_end:
                got[t] = dz[t - c.tok_begin].float().cpu().numpy()

    sp.run(target, lo, lr, lref, consume=consume)
    torch.cuda.synchronize()
    sp.check_status()
    L = layout
    # advantages and group validity (exact decision)
    A, ok = O.advantages(L.traj_reward, L.traj_group, L.traj_step_off, L.G)
    assert np.array_equal(sp.group_ok.cpu().numpy()[:L.G], ok)
    # selection: the oracle's rule on the GPU's own fp32 step entropies
    g = sp.gathered.cpu().numpy()
    rso = sp.rank_step_off.cpu().numpy()
    H_step = np.empty(L.S)
    for v in range(len(rso) - 1):
        H_step[rso[v]:rso[v + 1]] = g[v * sp.S_pad: v * sp.S_pad + (rso[v + 1] - rso[v])]
    keep_same, _ = O.select_steps(H_step.astype(np.float32).astype(np.float64), L.traj_group, L.traj_step_off,
                                  ok.astype(np.uint8), L.G, cfgf["entropy_q"], cfgf["select_rule"])
    keep = sp.keep.cpu().numpy()[:L.S]
    assert np.array_equal(keep, keep_same)
    for gi in range(L.G):                            # >= 80% of every valid group's steps kept
        steps = np.arange(L.traj_step_off[gi * 8], L.traj_step_off[(gi + 1) * 8])
        if ok[gi]:
            assert keep[steps].sum() >= np.ceil(0.8 * len(steps))
    tok_keep = np.repeat(keep, np.diff(L.step_tok_off)).astype(bool)
    inv_norm = 1.0 / float(tok_keep.sum())
    nd = sp.norm.cpu().numpy()
    assert nd[0] == tok_keep.sum()
    s_of_t = O.step_of_token(L.step_tok_off, T)
    tr_of_s = O.traj_of_step(L.traj_step_off, L.S)
    pool = [sp.pool_logits[k] for k in range(P)]
    for t, ci in zip(sample, chunk_of):
        c = sp.chunks[ci]
        st = sp.state[ci]
        r_loc = t - c.tok_begin
        z = pool[ci % P][r_loc].float().cpu().numpy()
        y = int(target[t])
        lse, logp, H, p = O.token_row(z, y)
        assert abs(float(st["lse"][r_loc]) - lse) <= RTOL_ENT * abs(lse) + ATOL_ENT
        assert abs(float(st["H"][r_loc]) - H) <= RTOL_ENT * H + ATOL_ENT
        assert abs(float(st["logp"][r_loc]) - logp) <= ATOL_LOGP
        ell, dell, w, r, clipped, kl = O.token_loss(logp, float(lo[t]), float(lr[t]), float(lref[t]),
                                                    A[tr_of_s[s_of_t[t]]], cfgf)
        if min(abs(r - (1 - cfgf["eps_low"])), abs(r - (1 + cfgf["eps_high"]))) < 1e-5 * r:
            continue
        assert abs(float(st["ell"][r_loc]) - ell) <= RTOL_TOK * abs(ell) + ATOL_TOK
        dz = got[t]
        if not tok_keep[t]:
            assert np.all(dz == 0)
            continue
        gg = inv_norm * dell
        onehot = np.zeros_like(p)
        onehot[y] = 1.0
        dref = gg * (onehot - p)
        dg = inv_norm * (RTOL_TOK * abs(dell) + ATOL_TOK)
        assert np.all(np.abs(dz - dref) <= grad_tol(dref, np.maximum(p, onehot), gg, dg, torch.bfloat16)), t
    # loss = inv_norm * sum of the GPU's own kept per-token terms (fp64)
    ell_all = np.concatenate([sp.state[i]["ell"][:c.T_loc].cpu().numpy() for i, c in enumerate(sp.chunks)])
    L_chk = np.sum(ell_all[tok_keep].astype(np.float64)) * inv_norm
    loss = sp.stats_dict()["loss"]
    assert abs(loss - L_chk) <= 1e-9 * np.sum(np.abs(ell_all[tok_keep])) * inv_norm + 1e-15
