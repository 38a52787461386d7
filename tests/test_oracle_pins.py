"""Pins of the float64 oracle to things other than itself (CPU only).

Every oracle function is checked against at least one of: a value the paper /
SPEC prints (tests/golden/*.json, each cited), a closed form, a textbook /
library special case, brute force on tiny inputs, central finite differences,
or an independent float64 torch-autograd derivation.  DESIGN.md §4 maps each
oracle function to its pins.
"""
import itertools
import math

import numpy as np
import pytest
import torch

from oracle import dart_oracle as O

E = math.e


# ------------------------------------------------------------------ constants
def test_paper_constants_are_the_oracle_defaults(golden):
    c = golden("paper_constants.json")
    assert O.DEFAULT_CFG["eps_low"] == c["eps_low"]["value"]
    assert O.DEFAULT_CFG["eps_high"] == c["eps_high"]["value"]
    assert O.DEFAULT_CFG["beta_kl"] == c["beta_kl"]["value"]
    assert O.DEFAULT_CFG["is_cap"] == c["is_cap"]["value"]
    assert O.DEFAULT_CFG["inv_temperature"] == 1.0 / c["temperature"]["value"]
    assert O.DEFAULT_CFG["entropy_q"] == c["entropy_q"]["value"]


# ------------------------------------------------------------------ P1 / P2 / P3
def test_p1_log_softmax_closed_form(golden):
    ex = golden("spec_examples.json")["softmax_p0_V4"]
    lse, logp, H, p = O.token_row(np.array([1.0, 0, 0, 0]), 0)
    assert abs(p[0] - ex["p0"]) < ex["tol"]
    assert abs(p[0] - E / (E + 3)) < 1e-15                 # closed form
    assert abs(lse - math.log(E + 3)) < 1e-15
    assert abs(logp - (1 - math.log(E + 3))) < 1e-15
    assert abs(p[1] - 1 / (E + 3)) < 1e-15


def test_p1_log_softmax_matches_library_on_random_rows():
    rng = np.random.default_rng(0)
    for V in (2, 7, 64, 1000):
        z = rng.normal(0, 3, V)
        y = int(rng.integers(0, V))
        for invT in (1.0, 0.5, 2.0):
            lse, logp, H, p = O.token_row(z, y, invT)
            zt = torch.tensor(z, dtype=torch.float64) * invT
            ref_lsm = torch.log_softmax(zt, 0)
            assert abs(lse - torch.logsumexp(zt, 0).item()) < 1e-12
            assert abs(logp - ref_lsm[y].item()) < 1e-12
            ref_H = torch.distributions.Categorical(logits=zt).entropy().item()
            assert abs(H - ref_H) < 1e-12 * max(1, abs(ref_H))
            assert np.allclose(p, torch.softmax(zt, 0).numpy(), rtol=1e-13, atol=0)


@pytest.mark.parametrize("V,H", [(16, 2.772588722), (512, 6.238324625), (152064, 11.932056764)])
def test_p2_uniform_entropy_is_lnV(V, H, golden):
    lse, logp, Ht, p = O.token_row(np.zeros(V), 3)
    assert abs(Ht - math.log(V)) < 1e-12 * math.log(V)
    assert abs(Ht - H) < 1e-9
    assert abs(logp + math.log(V)) < 1e-12
    if V == 16:
        ex = golden("spec_examples.json")["uniform_entropy_V16"]
        assert abs(Ht - ex["H"]) < ex["tol"]


def test_p2_entropy_V4_closed_form():
    _, _, H, _ = O.token_row(np.array([1.0, 0, 0, 0]), 0)
    # H = log(e+3) - e/(e+3)  (p0 = e/(e+3), p_i = 1/(e+3))
    assert abs(H - (math.log(E + 3) - E / (E + 3))) < 1e-15
    assert abs(H - 1.2683014942) < 1e-10


def test_p3_one_hot_rows():
    z = np.array([0.0, -np.inf, -np.inf, -np.inf, -np.inf])
    lse, logp, H, p = O.token_row(z, 0)
    assert H == 0.0 and logp == 0.0 and lse == 0.0
    assert p[0] == 1.0 and np.all(p[1:] == 0)
    # gradient of a one-hot row is exactly zero (onehot - p = 0)
    b = dict(logits=z[None, :], target=[0], logp_old=[-0.1], logp_rollout=[-0.1], logp_ref=[0.0],
             traj_group=[0, 0], traj_reward=[1.0, 0.0], traj_step_off=[0, 1, 1], step_tok_off=[0, 1], G=1)
    # (second trajectory has zero steps -> group still has one step; sigma=0 -> skipped)
    out = O.loss_pass(b, dict(norm_mode=O.NORM_SUM, adv_eps=1e-3))
    assert np.all(out["dz"][0] == 0)
    # near one-hot with finite logits: tiny but positive entropy (abs floor of Q16)
    z = np.zeros(16)
    z[5] = 30.0
    _, logp, H, _ = O.token_row(z, 5)
    assert 0 < H < 1e-8
    assert -1e-11 < logp <= 0


def test_entropy_bounds_and_uniform_iff():
    rng = np.random.default_rng(1)
    for _ in range(200):
        V = int(rng.integers(2, 300))
        z = rng.normal(0, rng.uniform(0.01, 10), V)
        _, _, H, _ = O.token_row(z, 0)
        assert -1e-15 <= H <= math.log(V) + 1e-12
        assert H < math.log(V) - 1e-12            # non-uniform => strictly below ln V


# ------------------------------------------------------------------ P4 advantages
def _adv(rewards, steps, adv_eps=0.0):
    off = np.concatenate([[0], np.cumsum(steps)])
    return O.advantages(rewards, np.zeros(len(rewards), dtype=np.int32), off, 1, adv_eps)


def test_p4_advantages_spec_examples(golden):
    ex = golden("spec_examples.json")
    e = ex["adv_step_rewards"]
    A, ok = _adv(e["traj_rewards"], e["traj_steps"])
    assert ok[0] == 1 and np.allclose(A, e["A"], atol=e["tol"], rtol=0)
    e = ex["adv_step_weighted"]
    A, ok = _adv(e["traj_rewards"], e["traj_steps"])
    assert np.allclose(A, e["A"], atol=e["tol"], rtol=0)
    # closed form: Rbar = 1/4, sigma = sqrt(3)/4 -> A = sqrt(3), -1/sqrt(3)
    assert abs(A[0] - math.sqrt(3)) < 1e-15 and abs(A[1] + 1 / math.sqrt(3)) < 1e-15
    e = ex["adv_all_equal"]
    A, ok = _adv(e["traj_rewards"], e["traj_steps"])
    assert ok[0] == e["group_ok"] and np.all(A == 0)
    # the flag adv_eps > 0 keeps the group (verl-style)
    A, ok = _adv(e["traj_rewards"], e["traj_steps"], adv_eps=1e-6)
    assert ok[0] == 1 and np.all(A == 0)
    # exact arithmetic: equal non-dyadic rewards over step counts whose float mean
    # does not round back to R still give R_bar = R and A = 0 exactly (not residue / eps)
    for r, steps in ((0.3, [3, 5, 7]), (0.1, [1, 2, 3, 4, 5, 6]), (0.7, [11])):
        A, ok = _adv([r] * len(steps), steps, adv_eps=1e-6)
        assert ok[0] == 1 and np.all(A == 0.0), (r, steps, A)


def test_p4_advantage_invariants_random_groups():
    rng = np.random.default_rng(2)
    for _ in range(100):
        G = int(rng.integers(1, 5))
        ntraj = rng.integers(1, 9, size=G)
        traj_group = np.repeat(np.arange(G), ntraj).astype(np.int32)
        steps = rng.integers(1, 12, size=len(traj_group))
        rew = rng.random(len(traj_group))
        off = np.concatenate([[0], np.cumsum(steps)])
        A, ok = O.advantages(rew, traj_group, off, G)
        for g in range(G):
            idx = np.nonzero(traj_group == g)[0]
            A_steps = np.repeat(A[idx], steps[idx])       # one entry per step of D
            if ok[g]:
                assert abs(A_steps.mean()) < 1e-9
                assert abs(A_steps.std() - 1.0) < 1e-9                # population std
                # A is an increasing affine function of R within the group
                order = np.argsort(rew[idx])
                assert np.all(np.diff(A[idx][order]) >= -1e-12)
            else:
                assert len(set(rew[idx])) == 1


def test_advantage_groups_are_independent():
    # two groups concatenated == each group alone
    A1, ok1 = _adv([1, 0, 0.5], [2, 1, 4])
    A2, ok2 = _adv([0.2, 0.9], [3, 3])
    off = np.concatenate([[0], np.cumsum([2, 1, 4, 3, 3])])
    A, ok = O.advantages([1, 0, 0.5, 0.2, 0.9], [0, 0, 0, 1, 1], off, 2)
    assert np.array_equal(A, np.concatenate([A1, A2])) and list(ok) == [1, 1]


# ------------------------------------------------------------------ step entropy
def test_step_entropy_spec_examples(golden):
    ex = golden("spec_examples.json")
    for k in ("step_entropy_mean", "step_entropy_zero"):
        e = ex[k]
        h = O.step_entropy(e["H_tok"], [0, len(e["H_tok"])])
        assert abs(h[0] - e["H_step"]) <= max(e["tol"], 1e-15)
    h = O.step_entropy([math.log(16)] * 2, [0, 2])
    assert abs(h[0] - 2.7726) < 1e-4


# ------------------------------------------------------------------ P5 selection
def test_p5_selection_spec_examples(golden):
    ex = golden("spec_examples.json")
    e = ex["gate_0p1_to_1p0"]
    assert abs(O.threshold(e["H"], e["q"]) - e["tau"]) < 1e-15
    for k in ("gate_0p1_to_1p0", "gate_all_equal", "gate_n1"):
        e = ex[k]
        n = len(e["H"])
        keep, tau = O.select_steps(e["H"], [0] * n, np.arange(n + 1), [1], 1, e["q"])
        assert int(keep.sum()) == e["kept"]


def _brute_keep(H, k):
    """Independent counting form of the order-statistic rule: step i is kept
    iff at least k+1 steps (itself included) have entropy <= H_i."""
    H = list(H)
    return [int(sum(1 for hj in H if hj <= hi) >= k + 1) for hi in H]


@pytest.mark.parametrize("rule", [O.SEL_FLOOR, O.SEL_CEIL])
def test_p5_selection_brute_force_ties_and_permutations(rule):
    q = 0.2
    for n in range(1, 7):
        k = math.floor(q * n) if rule == O.SEL_FLOOR else min(math.ceil(q * n), n - 1)
        # every tie pattern (values from a set of size <= n) and every ordering
        for vals in itertools.product(range(n), repeat=n):
            H = [0.1 * v for v in vals]
            keep, tau = O.select_steps(H, [0] * n, np.arange(n + 1), [1], 1, q, rule)
            assert list(keep) == _brute_keep(H, k), (H, rule)


def test_p5_kept_counts_table():
    # kept counts, n = 1..12, distinct values
    want = {O.SEL_FLOOR: [1, 2, 3, 4, 4, 5, 6, 7, 8, 8, 9, 10],
            O.SEL_CEIL: [1, 1, 2, 3, 4, 4, 5, 6, 7, 8, 8, 9],
            O.SEL_LINEAR: [1, 1, 2, 3, 4, 5, 5, 6, 7, 8, 9, 9]}
    for rule, counts in want.items():
        for n in range(1, 13):
            H = np.arange(n) * 0.37 + 0.1
            keep, _ = O.select_steps(H, [0] * n, np.arange(n + 1), [1], 1, 0.2, rule)
            assert int(keep.sum()) == counts[n - 1], (rule, n)
            if rule == O.SEL_FLOOR:
                assert keep.sum() == math.ceil(0.8 * n - 1e-12)     # "top 80%"


def test_p5_linear_rule_is_torch_quantile():
    rng = np.random.default_rng(3)
    for _ in range(200):
        n = int(rng.integers(1, 40))
        H = rng.random(n)
        q = float(rng.random())
        tau = O.threshold(H, q, O.SEL_LINEAR)
        ref = torch.quantile(torch.tensor(H, dtype=torch.float64), q, interpolation="linear").item()
        assert abs(tau - ref) < 1e-14


def test_p5_selection_invariants_random():
    rng = np.random.default_rng(4)
    for _ in range(300):
        n = int(rng.integers(1, 60))
        H = np.round(rng.random(n), int(rng.integers(1, 4)))       # ties
        q = float(rng.choice([0.0, 0.1, 0.2, 0.5, 0.9]))
        keep, tau = O.select_steps(H, [0] * n, np.arange(n + 1), [1], 1, q)
        assert keep.sum() >= math.ceil((1 - q) * n - 1e-9)
        assert np.all(H[keep.astype(bool)] >= tau[0])
        assert np.all(H[~keep.astype(bool)] < tau[0])
        # group_ok = 0 masks the whole group
        keep0, _ = O.select_steps(H, [0] * n, np.arange(n + 1), [0], 1, q)
        assert keep0.sum() == 0
        # OFF keeps everything
        keep1, _ = O.select_steps(H, [0] * n, np.arange(n + 1), [1], 1, q, O.SEL_OFF)
        assert keep1.sum() == n


def test_selection_is_per_group():
    H = [0.1, 0.2, 0.3, 5.0, 6.0, 7.0, 8.0]
    # traj 0 (group 0): steps 0..2 ; traj 1 (group 1): steps 3..6
    keep, tau = O.select_steps(H, [0, 1], [0, 3, 7], [1, 1], 2, 0.5)
    assert list(keep) == [0, 1, 1, 0, 0, 1, 1]
    assert list(tau) == [0.2, 7.0]


# ------------------------------------------------------------------ P6 / P7 scalar terms
def test_p6_is_weight(golden):
    ex = golden("spec_examples.json")
    e = ex["is_equal"]
    assert O.is_weight(e["logp_old"], e["logp_roll"], e["C"]) == e["w"]
    e = ex["is_truncated"]
    assert O.is_weight(e["log_ratio"], 0.0, e["C"]) == e["w"]
    e = ex["is_half"]
    assert abs(O.is_weight(math.log(e["ratio"]), 0.0, e["C"]) - e["w"]) <= e["tol"]
    rng = np.random.default_rng(5)
    for _ in range(1000):
        a, b, C = rng.normal(0, 3), rng.normal(0, 3), rng.uniform(0.1, 3)
        w = O.is_weight(a, b, C)
        assert 0 <= w <= C


def test_p7_surrogate(golden):
    ex = golden("spec_examples.json")
    for k in ("surrogate_clip_hi", "surrogate_clip_lo"):
        e = ex[k]
        assert abs(O.surrogate(e["r"], e["A"], e["eps_low"], e["eps_high"]) - e["value"]) <= e["tol"]
        assert O.surrogate_dlogp(e["r"], e["A"], e["eps_low"], e["eps_high"]) == 0.0
    # inside the trust region the surrogate is r*A, derivative A*r
    assert O.surrogate(1.1, -2.0, 0.2, 0.28) == 1.1 * -2.0
    assert O.surrogate_dlogp(1.1, -2.0, 0.2, 0.28) == -2.0 * 1.1
    # the "other side" is never clipped by min(): A>0, r<1-eps keeps r*A
    assert O.surrogate(0.5, 1.0, 0.2, 0.28) == 0.5
    assert O.surrogate_dlogp(0.5, 1.0, 0.2, 0.28) == 0.5
    # clip bound (SPEC trainer invariant): surrogate <= (1+eps_high) A for A>0
    rng = np.random.default_rng(6)
    for _ in range(1000):
        r, A = rng.uniform(0, 3), rng.normal()
        s = O.surrogate(r, A, 0.2, 0.28)
        if A > 0:
            assert s <= (1.28) * A + 1e-15
        assert s <= r * A + 1e-15


def test_k3_kl():
    assert O.kl_k3(-1.0, -1.0) == 0.0 and O.kl_k3_dlogp(-1.0, -1.0) == 0.0
    rng = np.random.default_rng(7)
    for _ in range(200):
        a, b = rng.normal(0, 2), rng.normal(0, 2)
        assert O.kl_k3(a, b) >= 0
        h = 1e-6
        fd = (O.kl_k3(a + h, b) - O.kl_k3(a - h, b)) / (2 * h)
        assert abs(fd - O.kl_k3_dlogp(a, b)) < 1e-6 * max(1, abs(fd))


# ------------------------------------------------------------------ P9 worked example
def _p9_batch(g, d_old, d_roll, d_ref=None):
    z = np.array(g["logits"], dtype=np.float64)
    logp = np.array([O.token_row(z[t], g["target"][t])[1] for t in range(4)])
    lo = logp + np.array(d_old)
    lr = lo + np.array(d_roll)
    lref = logp + (np.array(d_ref) if d_ref is not None else 0.0)
    return dict(logits=z, target=g["target"], logp_old=lo, logp_rollout=lr, logp_ref=lref,
                traj_group=g["traj_group"], traj_reward=g["traj_reward"],
                traj_step_off=g["traj_step_off"], step_tok_off=g["step_tok_off"], G=1)


def test_p9_intermediates(golden):
    g = golden("p9_worked_example.json")
    b = _p9_batch(g, [0] * 4, [0] * 4)
    out = O.loss_pass(b, dict(entropy_q=0.2, beta_kl=0.0, is_cap=1.0))
    tol = g["tol"]
    assert np.allclose(out["lse"], g["lse"], atol=tol, rtol=0)
    assert np.allclose(out["H"], g["H_tok"], atol=tol, rtol=0)
    assert np.allclose(out["logp"], g["logp"], atol=tol, rtol=0)
    assert np.allclose(out["step_H"], g["H_step"], atol=tol, rtol=0)
    assert np.allclose(out["A_traj"], g["A_traj"], atol=tol, rtol=0)
    assert abs(out["A_traj"][0] - math.sqrt(2)) < 1e-15                # closed form
    assert abs(out["A_traj"][1] + 1 / math.sqrt(2)) < 1e-15
    assert abs(out["tau"][0] - g["tau_q0.2"]) < tol and list(out["keep"]) == g["keep_q0.2"]
    out = O.loss_pass(b, dict(entropy_q=0.5, beta_kl=0.0))
    assert abs(out["tau"][0] - g["tau_q0.5"]) < tol and list(out["keep"]) == g["keep_q0.5"]
    # closed forms of row 2 (z = [2,1,0,-1]): lse = log(e^2+e+1+e^-1)
    assert abs(out["lse"][2] - math.log(E ** 2 + E + 1 + 1 / E)) < 1e-14


def test_p9_loss_and_gradient_C1_C2(golden):
    g = golden("p9_worked_example.json")
    run = g["run"]
    b = _p9_batch(g, run["d_old"], run["d_roll"])
    out = O.loss_pass(b, dict(entropy_q=run["q"], beta_kl=0.0, is_cap=1.0))
    c = g["C1"]
    assert np.allclose(out["w"], c["w"], atol=1e-10, rtol=0)
    assert np.allclose(out["r"], c["r"], atol=1e-10, rtol=0)
    assert np.allclose(out["ell"], c["ell"], atol=1e-10, rtol=0)
    assert abs(out["loss"] - c["loss"]) < 1e-12
    # hand derivation: ell_0 = -e^-0.1 sqrt2, ell_1 = -e^-0.5 * 1.28 sqrt2 (clipped),
    # ell_2 = +1/sqrt2, token mean over the 3 kept tokens
    L = (-math.exp(-0.1) * math.sqrt(2) - math.exp(-0.5) * 1.28 * math.sqrt(2) + 1 / math.sqrt(2)) / 3
    assert abs(out["loss"] - L) < 1e-14
    assert np.allclose(out["dz"][0], c["dz_t0"], atol=1e-10, rtol=0)
    assert np.allclose(out["dz"][2], c["dz_t2"], atol=1e-10, rtol=0)
    assert np.all(out["dz"][1] == 0) and np.all(out["dz"][3] == 0)     # clipped / masked
    out2 = O.loss_pass(b, dict(entropy_q=run["q"], beta_kl=0.0, is_cap=2.0))
    assert abs(out2["w"][2] - g["C2"]["w2"]) < 1e-10   # w of token t2 = e^0.2
    assert abs(out2["loss"] - g["C2"]["loss"]) < 1e-12
    assert np.allclose(out2["dz"][2], g["C2"]["dz_t2"], atol=1e-10, rtol=0)


def test_p9_kl_variant(golden):
    g = golden("p9_worked_example.json")
    run, k = g["run"], g["KL"]
    b = _p9_batch(g, run["d_old"], run["d_roll"], k["d_ref"])
    out = O.loss_pass(b, dict(entropy_q=run["q"], beta_kl=k["beta"], is_cap=k["C"]))
    assert np.allclose(out["kl"], k["k3"], atol=1e-8, rtol=0)
    assert abs(out["loss"] - k["loss_token_mean"]) < 1e-12
    assert np.allclose(out["dz"][1], k["dz_t1_token_mean"], atol=1e-8, rtol=0)
    out = O.loss_pass(b, dict(entropy_q=run["q"], beta_kl=k["beta"], is_cap=k["C"],
                              norm_mode=O.NORM_STEP_MEAN_KEPT))
    assert abs(out["loss"] - k["loss_step_mean"]) < 1e-12
    # closed form of k3 for d = -0.2
    assert abs(out["kl"][0] - (math.exp(-0.2) + 0.2 - 1)) < 1e-15


# ------------------------------------------------------------------ P8 on-policy identity
def test_p8_on_policy_identity():
    rng = np.random.default_rng(8)
    T, V = 12, 9
    z = rng.normal(0, 2, (T, V))
    y = rng.integers(0, V, T)
    logp = np.array([O.token_row(z[t], y[t])[1] for t in range(T)])
    b = dict(logits=z, target=y, logp_old=logp.copy(), logp_rollout=logp - 0.05 * rng.random(T),
             logp_ref=logp, traj_group=[0, 0, 0], traj_reward=[1.0, 0.0, 0.3],
             traj_step_off=[0, 2, 3, 5], step_tok_off=[0, 2, 4, 7, 9, 12], G=1)
    out = O.loss_pass(b, dict(entropy_q=0.0, beta_kl=0.1))
    assert np.allclose(out["r"], 1.0, rtol=0, atol=1e-15)
    assert np.allclose(out["kl"], 0.0, atol=1e-15)
    # surrogate reduces to the unclipped objective: ell = -w A, dell = -w A
    assert np.allclose(out["ell"], -out["w"] * out["A_tok"], atol=1e-14)
    assert np.allclose(out["dell"], -out["w"] * out["A_tok"], atol=1e-14)
    kt = out["keep"][O.step_of_token(b["step_tok_off"], T)].astype(bool)
    assert abs(out["loss"] - np.sum(-out["w"][kt] * out["A_tok"][kt]) / kt.sum()) < 1e-14


# ------------------------------------------------------------------ P10 / P11 gradients
def _random_batch(rng, V, G=2, beta=0.1):
    ntraj = rng.integers(2, 4, size=G)
    traj_group = np.repeat(np.arange(G), ntraj)
    steps = rng.integers(1, 4, size=len(traj_group))
    traj_step_off = np.concatenate([[0], np.cumsum(steps)])
    S = int(traj_step_off[-1])
    ntok = rng.integers(1, 4, size=S)
    step_tok_off = np.concatenate([[0], np.cumsum(ntok)])
    T = int(step_tok_off[-1])
    z = rng.normal(0, 2, (T, V))
    y = rng.integers(0, V, T)
    logp = np.array([O.token_row(z[t], y[t])[1] for t in range(T)])
    lo = logp + rng.normal(0, 0.3, T)
    return dict(logits=z, target=y, logp_old=lo, logp_rollout=lo + rng.normal(0, 0.3, T),
                logp_ref=logp + rng.normal(0, 0.2, T), traj_group=traj_group,
                traj_reward=rng.random(len(traj_group)), traj_step_off=traj_step_off,
                step_tok_off=step_tok_off, G=G)


@pytest.mark.parametrize("mode", [O.NORM_TOKEN_MEAN_KEPT, O.NORM_STEP_MEAN_KEPT, O.NORM_SUM,
                                  O.NORM_TOKEN_MEAN_ALL, O.NORM_STEP_MEAN_ALL])
@pytest.mark.parametrize("invT", [1.0, 0.7])
@pytest.mark.parametrize("ratio", [O.RATIO_TOKEN, O.RATIO_STEP])
def test_p10_finite_differences(mode, invT, ratio):
    rng = np.random.default_rng(10 + mode)
    b = _random_batch(rng, V=7)
    cfg = dict(entropy_q=0.3, beta_kl=0.1, is_cap=1.0, norm_mode=mode, inv_temperature=invT, ratio_level=ratio)
    out = O.loss_pass(b, cfg)
    keep = out["keep"]
    h = 1e-6
    z0 = b["logits"]
    for t in range(z0.shape[0]):
        for v in range(z0.shape[1]):
            zp, zm = z0.copy(), z0.copy()
            zp[t, v] += h
            zm[t, v] -= h
            Lp = O.loss_pass({**b, "logits": zp}, cfg, keep_override=keep, want_grad=False)["loss"]
            Lm = O.loss_pass({**b, "logits": zm}, cfg, keep_override=keep, want_grad=False)["loss"]
            fd = (Lp - Lm) / (2 * h)
            an = out["dz"][t][v]
            # skip coordinates sitting on a clip boundary (non-differentiable)
            r = out["r"][t]
            if min(abs(r - 0.8), abs(r - 1.28)) < 1e-4:
                continue
            assert abs(fd - an) <= 1e-6 * max(1e-3, abs(an)) + 1e-9, (t, v, fd, an)


def test_p10_gradient_matches_torch_autograd():
    """Independent derivation: float64 torch autograd through log_softmax /
    gather / minimum / clamp, with the oracle's mask and step weights."""
    rng = np.random.default_rng(11)
    for trial in range(5):
        b = _random_batch(rng, V=int(rng.integers(3, 40)), G=3)
        cfg = dict(entropy_q=0.2, beta_kl=float(rng.choice([0.0, 0.1])), is_cap=float(rng.choice([1.0, 2.0])),
                   inv_temperature=float(rng.choice([1.0, 0.8])))
        out = O.loss_pass(b, cfg)
        c = {**O.DEFAULT_CFG, **cfg}
        z = torch.tensor(b["logits"], dtype=torch.float64, requires_grad=True)
        y = torch.tensor(b["target"])
        lsm = torch.log_softmax(z * c["inv_temperature"], -1)
        logp = lsm.gather(1, y[:, None])[:, 0]
        lo = torch.tensor(b["logp_old"])
        lr = torch.tensor(b["logp_rollout"])
        lref = torch.tensor(b["logp_ref"])
        A = torch.tensor(out["A_tok"])
        w = torch.clamp(torch.exp(lo - lr), max=c["is_cap"])
        r = torch.exp(logp - lo)
        sur = torch.minimum(r * A, torch.clamp(r, 1 - c["eps_low"], 1 + c["eps_high"]) * A)
        d = lref - logp
        ell = -w * sur + c["beta_kl"] * (torch.exp(d) - d - 1)
        L = torch.sum(torch.tensor(out["c_tok"]) * ell)
        L.backward()
        assert abs(L.item() - out["loss"]) < 1e-13
        for t, dz in out["dz"].items():
            assert np.allclose(z.grad[t].numpy(), dz, rtol=1e-12, atol=1e-15), (trial, t)


def test_step_ratio_gradient_matches_torch_autograd():
    """Step-level ratio: autograd of an independent float64
    torch expression with per-step sequence log-ratios."""
    rng = np.random.default_rng(21)
    for trial in range(5):
        b = _random_batch(rng, V=int(rng.integers(3, 30)), G=3)
        cfg = dict(entropy_q=0.2, beta_kl=float(rng.choice([0.0, 0.1])), is_cap=float(rng.choice([1.0, 2.0])),
                   ratio_level=O.RATIO_STEP, norm_mode=int(rng.integers(0, 5)))
        out = O.loss_pass(b, cfg)
        c = {**O.DEFAULT_CFG, **cfg}
        z = torch.tensor(b["logits"], dtype=torch.float64, requires_grad=True)
        logp = torch.log_softmax(z, -1).gather(1, torch.tensor(b["target"])[:, None])[:, 0]
        lo, lr, lref = (torch.tensor(b[k]) for k in ("logp_old", "logp_rollout", "logp_ref"))
        off = b["step_tok_off"]
        L = torch.zeros((), dtype=torch.float64)
        c_step = O.step_weights(out["keep"], off, c["norm_mode"], per_step_loss=True)
        for s_ in range(len(off) - 1):
            sl = slice(off[s_], off[s_ + 1])
            A = float(out["A_tok"][off[s_]])
            r = torch.exp(torch.sum(logp[sl] - lo[sl]))
            w = torch.clamp(torch.exp(torch.sum(lo[sl] - lr[sl])), max=c["is_cap"])
            sur = torch.minimum(r * A, torch.clamp(r, 1 - c["eps_low"], 1 + c["eps_high"]) * A)
            d = lref[sl] - logp[sl]
            L = L + c_step[s_] * (-w * sur + c["beta_kl"] * torch.sum(torch.exp(d) - d - 1))
        L.backward()
        assert abs(L.item() - out["loss"]) < 1e-13 * max(1.0, abs(L.item()))
        for t, dz in out["dz"].items():
            assert np.allclose(z.grad[t].numpy(), dz, rtol=1e-11, atol=1e-15), (trial, t)


def test_step_ratio_p9_closed_form(golden):
    """P9 example in step-ratio mode: step 0 = {t0, t1} of the success
    (A = sqrt2): log r = -0.1 + 0.3 = 0.2 (inside the clip range), log w =
    0 - 0.5; step 1 = {t2} (A = -1/sqrt2): r = 1, w = min(e^0.2, 1) = 1;
    step 2 masked (q = 0.5)."""
    g = golden("p9_worked_example.json")
    run = g["run"]
    b = _p9_batch(g, run["d_old"], run["d_roll"])
    l0 = -math.exp(-0.5) * math.exp(0.2) * math.sqrt(2)
    l1 = 1 / math.sqrt(2)
    out = O.loss_pass(b, dict(entropy_q=run["q"], beta_kl=0.0, is_cap=1.0, ratio_level=O.RATIO_STEP))
    assert abs(out["loss"] - (l0 + l1) / 3) < 1e-14              # token-mean: N_keep_tok = 3
    out = O.loss_pass(b, dict(entropy_q=run["q"], beta_kl=0.0, is_cap=1.0, ratio_level=O.RATIO_STEP,
                              norm_mode=O.NORM_STEP_MEAN_KEPT))
    assert abs(out["loss"] - (l0 + l1) / 2) < 1e-14              # step-mean: N_keep_step = 2
    # every token of step 0 gets the same surrogate gradient -w A r
    assert abs(out["dell"][0] - out["dell"][1]) < 1e-15
    assert abs(out["dell"][0] - (-math.exp(-0.5) * math.sqrt(2) * math.exp(0.2))) < 1e-14


def test_p11_uniform_row_gradient():
    V = 16
    b = dict(logits=np.zeros((2, V)), target=[3, 4], logp_old=[-math.log(V) + 0.05, -math.log(V)],
             logp_rollout=[-math.log(V), -math.log(V)], logp_ref=[-math.log(V)] * 2,
             traj_group=[0, 0], traj_reward=[1.0, 0.0], traj_step_off=[0, 1, 2], step_tok_off=[0, 1, 2], G=1)
    out = O.loss_pass(b, dict(entropy_q=0.0, beta_kl=0.0, norm_mode=O.NORM_SUM, inv_temperature=0.5))
    for t in range(2):
        g = out["c_tok"][t] * out["dell"][t]
        want = 0.5 * g * (np.eye(V)[b["target"][t]] - 1.0 / V)
        assert np.allclose(out["dz"][t], want, atol=1e-16, rtol=1e-14)


# ------------------------------------------------------------------ P12 invariants
def test_p12_invariants_random_batches():
    rng = np.random.default_rng(12)
    for _ in range(10):
        V = int(rng.integers(2, 64))
        b = _random_batch(rng, V=V, G=3)
        out = O.loss_pass(b, dict(entropy_q=0.2, is_cap=1.0))
        assert np.all(out["H"] >= 0) and np.all(out["H"] <= math.log(V) + 1e-12)
        assert np.all(out["w"] >= 0) and np.all(out["w"] <= 1.0)
        for t, dz in out["dz"].items():
            assert abs(dz.sum()) < 1e-15 * V + 1e-16          # softmax gradient sums to 0
        # kept fraction per valid group >= 1 - q
        off = b["traj_step_off"]
        for gi in range(b["G"]):
            steps = np.concatenate([np.arange(off[i], off[i + 1]) for i in np.nonzero(b["traj_group"] == gi)[0]])
            if out["group_ok"][gi]:
                assert out["keep"][steps].sum() >= math.ceil(0.8 * len(steps) - 1e-9)
            else:
                assert out["keep"][steps].sum() == 0


def test_norm_modes_closed_form():
    keep = np.array([1, 0, 1, 1], dtype=np.uint8)
    off = np.array([0, 2, 5, 6, 10])          # n = 2,3,1,4
    c = O.step_weights(keep, off, O.NORM_TOKEN_MEAN_KEPT)
    assert np.allclose(c, [1 / 7, 0, 1 / 7, 1 / 7])
    c = O.step_weights(keep, off, O.NORM_STEP_MEAN_KEPT)
    assert np.allclose(c, [1 / (3 * 2), 0, 1 / (3 * 1), 1 / (3 * 4)])
    c = O.step_weights(keep, off, O.NORM_TOKEN_MEAN_ALL)
    assert np.allclose(c, [1 / 10, 0, 1 / 10, 1 / 10])
    c = O.step_weights(keep, off, O.NORM_STEP_MEAN_ALL)
    assert np.allclose(c, [1 / 8, 0, 1 / 4, 1 / 16])
    c = O.step_weights(keep, off, O.NORM_SUM)
    assert np.allclose(c, [1, 0, 1, 1])
    assert np.all(O.step_weights(np.zeros(4, np.uint8), off, O.NORM_TOKEN_MEAN_KEPT) == 0)


# ------------------------------------------------------------------ exact KL
def test_exact_kl_spec_example_and_gibbs(golden):
    e = golden("spec_examples.json")["kl_exact_V2"]
    kl, _ = O.kl_exact_row(np.log(e["p_a"]), np.log(e["p_b"]))
    assert abs(kl - e["kl"]) < e["tol"]
    assert abs(kl - (0.9 * math.log(0.9 / 0.5) + 0.1 * math.log(0.1 / 0.5))) < 1e-15   # closed form
    rng = np.random.default_rng(30)
    for _ in range(300):
        V = int(rng.integers(2, 50))
        z, zr = rng.normal(0, 2, V), rng.normal(0, 2, V)
        kl, _ = O.kl_exact_row(z, zr)
        assert kl >= -1e-15                                             # Gibbs
        ref = torch.nn.functional.kl_div(torch.log_softmax(torch.tensor(zr), 0),
                                         torch.log_softmax(torch.tensor(z), 0), log_target=True,
                                         reduction="sum").item()
        assert abs(kl - ref) < 1e-12 * max(1.0, abs(ref))               # library routine
        assert O.kl_exact_row(z, z + 3.0)[0] < 1e-13                    # shift-invariant: identical -> 0


def _with_ref(b, rng, scale=0.3):
    b = dict(b)
    b["ref_logits"] = b["logits"] + rng.normal(0, scale, b["logits"].shape)
    return b


@pytest.mark.parametrize("ratio", [O.RATIO_TOKEN, O.RATIO_STEP])
def test_exact_kl_finite_differences(ratio):
    rng = np.random.default_rng(31)
    b = _with_ref(_random_batch(rng, V=6), rng)
    cfg = dict(entropy_q=0.3, beta_kl=0.3, is_cap=1.0, kl_mode=O.KL_EXACT, ratio_level=ratio, inv_temperature=0.8)
    out = O.loss_pass(b, cfg)
    h = 1e-6
    z0 = b["logits"]
    for t in range(z0.shape[0]):
        for v in range(z0.shape[1]):
            zp, zm = z0.copy(), z0.copy()
            zp[t, v] += h
            zm[t, v] -= h
            Lp = O.loss_pass({**b, "logits": zp}, cfg, keep_override=out["keep"], want_grad=False)["loss"]
            Lm = O.loss_pass({**b, "logits": zm}, cfg, keep_override=out["keep"], want_grad=False)["loss"]
            fd = (Lp - Lm) / (2 * h)
            an = out["dz"][t][v]
            if min(abs(out["r"][t] - 0.8), abs(out["r"][t] - 1.28)) < 1e-4:
                continue
            assert abs(fd - an) <= 1e-6 * max(1e-3, abs(an)) + 1e-9, (t, v, fd, an)


def test_exact_kl_gradient_matches_torch_autograd():
    rng = np.random.default_rng(32)
    for trial in range(4):
        b = _with_ref(_random_batch(rng, V=int(rng.integers(3, 30)), G=3), rng, 0.5)
        cfg = dict(entropy_q=0.2, beta_kl=0.1, is_cap=1.0, kl_mode=O.KL_EXACT)
        out = O.loss_pass(b, cfg)
        c = {**O.DEFAULT_CFG, **cfg}
        z = torch.tensor(b["logits"], dtype=torch.float64, requires_grad=True)
        lsm = torch.log_softmax(z, -1)
        lsq = torch.log_softmax(torch.tensor(b["ref_logits"]), -1)
        logp = lsm.gather(1, torch.tensor(b["target"])[:, None])[:, 0]
        lo, lr = torch.tensor(b["logp_old"]), torch.tensor(b["logp_rollout"])
        A = torch.tensor(out["A_tok"])
        w = torch.clamp(torch.exp(lo - lr), max=c["is_cap"])
        r = torch.exp(logp - lo)
        sur = torch.minimum(r * A, torch.clamp(r, 1 - c["eps_low"], 1 + c["eps_high"]) * A)
        kl = torch.sum(torch.exp(lsm) * (lsm - lsq), dim=-1)
        L = torch.sum(torch.tensor(out["c_tok"]) * (-w * sur + c["beta_kl"] * kl))
        L.backward()
        assert abs(L.item() - out["loss"]) < 1e-13
        for t, dz in out["dz"].items():
            assert np.allclose(z.grad[t].numpy(), dz, rtol=1e-11, atol=1e-15), (trial, t)


# ------------------------------------------------------------------ LM head
def test_lmhead_logits_brute_force_integers():
    """z_{t,v} = sum_k h_{t,k} W_{v,k}: integer inputs make every sum exact, so
    a pure-Python triple loop is the ground truth (catches a transposed W or a
    dropped index)."""
    rng = np.random.default_rng(40)
    T, V, d = 3, 5, 7
    h = rng.integers(-3, 4, (T, d)).astype(np.float64)
    W = rng.integers(-3, 4, (V, d)).astype(np.float64)
    z = O.lmhead_logits(h, W)
    assert z.shape == (T, V)
    for t in range(T):
        for v in range(V):
            acc = 0
            for k in range(d):
                acc += int(h[t, k]) * int(W[v, k])
            assert z[t, v] == acc


def test_lmhead_logits_special_cases():
    rng = np.random.default_rng(41)
    h = rng.normal(size=(4, 6))
    # W = first rows of the identity: the logits are the hidden coordinates
    assert np.array_equal(O.lmhead_logits(h, np.eye(6)[:3]), h[:, :3])
    # a single hot row picks one coordinate; a zero W gives uniform softmax (H = log V)
    W = np.zeros((5, 6))
    W[2, 4] = 1.0
    assert np.array_equal(O.lmhead_logits(h, W)[:, 2], h[:, 4])
    z0 = O.lmhead_logits(h, np.zeros((9, 6)))
    lse, logp, H, p = O.token_row(z0[0], 3)
    assert abs(H - math.log(9)) < 1e-14 and abs(logp + math.log(9)) < 1e-14


def test_lmhead_grads_match_torch_autograd_through_the_head():
    """dh = dz W and dW = dz^T h against float64 torch autograd of the whole
    loss composed with z = h W^T (an independent derivation: torch's own
    matmul backward and our loss written as torch ops)."""
    rng = np.random.default_rng(42)
    b = _random_batch(rng, V=6)
    T = len(b["target"])
    d = 5
    h = rng.normal(0, 1, (T, d))
    W = rng.normal(0, 0.7, (6, d))
    b = dict(b)
    b["logits"] = O.lmhead_logits(h, W)
    cfg = dict(entropy_q=0.3, beta_kl=0.1, is_cap=1.5, inv_temperature=0.9)
    out = O.loss_pass(b, cfg)
    dz = np.stack([out["dz"][t] for t in range(T)])
    dh, dW = O.lmhead_grads(dz, h, W)
    c = {**O.DEFAULT_CFG, **cfg}
    ht = torch.tensor(h, requires_grad=True)
    Wt = torch.tensor(W, requires_grad=True)
    z = ht @ Wt.T
    logp = torch.log_softmax(z * c["inv_temperature"], -1).gather(1, torch.tensor(b["target"])[:, None])[:, 0]
    lo, lr, lref = (torch.tensor(b[k]) for k in ("logp_old", "logp_rollout", "logp_ref"))
    A = torch.tensor(out["A_tok"])
    w = torch.clamp(torch.exp(lo - lr), max=c["is_cap"])
    r = torch.exp(logp - lo)
    sur = torch.minimum(r * A, torch.clamp(r, 1 - c["eps_low"], 1 + c["eps_high"]) * A)
    dd = lref - logp
    L = torch.sum(torch.tensor(out["c_tok"]) * (-w * sur + c["beta_kl"] * (torch.exp(dd) - dd - 1)))
    L.backward()
    assert abs(L.item() - out["loss"]) < 1e-12
    assert np.allclose(dh, ht.grad.numpy(), rtol=1e-10, atol=1e-13)
    assert np.allclose(dW, Wt.grad.numpy(), rtol=1e-10, atol=1e-13)
