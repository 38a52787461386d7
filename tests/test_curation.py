"""SURVEY §8(f) #4 (second half): host-side data curation, §4.1-4.2.

* the oracle (oracle/curation_oracle.py) pinned against what the paper states
  (8 rollouts at low success, fewer above 0.6; caps between 10 and 50 steps
  from successful lengths; at least one positive trajectory per task after
  pool injection) and hand-worked cases;
* the library's host functions (dart_rollout_counts / dart_trajectory_caps /
  dart_curate_batch) bit-exact against the oracle on seeded inputs;
* (gpu) the loss pass over a curated batch against the loss oracle.
CPU tests need only the built library (host code, no GPU)."""
import math

import numpy as np
import pytest

from oracle import curation_oracle as CO
from paper_2509_23866_b200 import build as B
from paper_2509_23866_b200 import synth


@pytest.fixture(scope="module")
def C():
    B.build()
    from paper_2509_23866_b200 import curation
    return curation


# ------------------------------------------------------------------ oracle pins
def test_rollout_count_paper_values():
    # "when a task achieves high success rates (above 0.6), we reduce its
    # rollout frequency from 8 to lower values ... low success rates maintain maximum sampling"
    assert CO.rollout_count(0, 0) == 8                      # no history: maximum sampling
    for ns, nt in [(0, 10), (3, 10), (6, 10), (3, 5)]:      # success rate <= 0.6 (3/5 exactly 0.6)
        assert CO.rollout_count(ns, nt) == 8
    assert CO.rollout_count(7, 10) < 8                      # above 0.6: fewer
    assert CO.rollout_count(10, 10) == CO.N_MIN == 2        # R15: n_min at success rate 1
    # R15 closed form: sr = 0.8 -> halfway -> 8 - round(0.5 * 6) = 5; sr = 0.7 -> 8 - round(1.5) = 6
    assert CO.rollout_count(8, 10) == 5
    assert CO.rollout_count(7, 10) == 6


def test_rollout_count_monotone_and_bounded():
    prev = 99
    for k in range(0, 1001):
        n = CO.rollout_count(k, 1000)
        assert CO.N_MIN <= n <= CO.N_MAX
        assert n <= prev
        prev = n
    assert all(CO.rollout_count(k, 1000, n_max=32, n_min=4) in range(4, 33) for k in range(1001))


def test_trajectory_cap_paper_values():
    # from the historical maximum successful length; "simple clicking
    # tasks might terminate after 10 steps, while complex ... can extend to 50 steps"
    assert CO.trajectory_cap(None) == 50 and CO.trajectory_cap(-1) == 50   # no success yet: explore
    assert CO.trajectory_cap(3) == 10
    assert CO.trajectory_cap(10) == 10
    assert CO.trajectory_cap(27) == 27
    assert CO.trajectory_cap(50) == 50
    assert CO.trajectory_cap(80) == 50


def test_curate_batch_hand_example():
    # task 0: one success, one over-long rollout (cap 3 -> cut, reward 0)
    # task 1: all fail, pool has 2 -> draw 0.75 picks index 1, appended
    # task 2: all fail, empty pool -> stays all-fail
    # task 3: no rollouts, no pool -> no group
    tasks = [[([5, 6], 1.0), ([1, 2, 3, 4], 1.0)],
             [([7], 0.0), ([8, 9], 0.2)],
             [([3], 0.0)],
             []]
    pool = [[], [([11], 1.0), ([12, 13], 1.0)], [], []]
    out = CO.curate_batch(tasks, caps=[3, 10, 10, 10], pool=pool, pool_draw=[0.0, 0.75, 0.5, 0.5])
    assert out["G"] == 3
    assert out["traj_group"] == [0, 0, 1, 1, 1, 2]
    assert out["traj_reward"] == [1.0, 0.0, 0.0, 0.2, 1.0, 0.0]
    assert out["traj_step_off"] == [0, 2, 5, 6, 8, 10, 11]
    assert out["step_tok_off"] == [0, 5, 11, 12, 14, 17, 24, 32, 41, 53, 66, 69]
    assert out["traj_source"] == [0, 1, 2, 3, -2, 4]


def _random_round(seed, G=24):
    d = synth.make_curation_inputs(G, seed=seed)
    n = [CO.rollout_count(int(a), int(b)) for a, b in zip(d["n_success"], d["n_total"])]
    caps = [CO.trajectory_cap(int(m)) for m in d["max_success_len"]]
    tasks = [d["make_rollouts"](n[g], d["p_succ"][g]) for g in range(G)]
    return d, n, caps, tasks


@pytest.mark.parametrize("seed", range(6))
def test_curate_batch_invariants(seed):
    d, n, caps, tasks = _random_round(seed)
    out = CO.curate_batch(tasks, caps, d["pool"], d["pool_draw"])
    tg, tr, tso, src = (np.asarray(out[k]) for k in ("traj_group", "traj_reward", "traj_step_off", "traj_source"))
    assert np.all(np.diff(tg) >= 0) and tg[0] == 0 and tg[-1] == out["G"] - 1      # contiguous groups
    assert np.all(np.diff(tso) >= 1)                                              # >= 1 step each
    assert np.all(np.diff(out["step_tok_off"]) >= 1)
    flat_pool = [tr_ for p in d["pool"] for tr_ in p]
    g_of_task = {}
    g_out = 0
    for g in range(len(tasks)):
        if tasks[g] or d["pool"][g]:
            g_of_task[g] = g_out
            g_out += 1
    for i in range(len(tg)):
        L = tso[i + 1] - tso[i]
        if src[i] >= 0:              # rollouts respect their task's cap
            gt = [g for g in range(len(tasks)) if sum(len(t) for t in tasks[:g]) <= src[i]
                  < sum(len(t) for t in tasks[:g + 1])][0]
            assert L <= caps[gt]
        else:
            steps, reward = flat_pool[-src[i] - 1]
            assert L == len(steps) and tr[i] == reward
    # every task with a non-empty pool holds at least one positive trajectory
    for g in range(len(tasks)):
        if d["pool"][g]:
            rows = tr[tg == g_of_task[g]]
            assert np.any(rows >= CO.SUCCESS_REWARD)
    assert len(tg) <= sum(len(t) for t in tasks) + len(tasks)


# ------------------------------------------------------------------ library vs oracle (host code)
@pytest.mark.parametrize("seed", range(8))
def test_library_rollout_counts_and_caps_match_oracle(C, seed):
    d = synth.make_curation_inputs(40, seed=seed)
    cfg = C.CurationConfig()
    n = C.rollout_counts(cfg, d["n_success"], d["n_total"])
    assert n.tolist() == [CO.rollout_count(int(a), int(b)) for a, b in zip(d["n_success"], d["n_total"])]
    caps = C.trajectory_caps(cfg, d["max_success_len"])
    assert caps.tolist() == [CO.trajectory_cap(int(m)) for m in d["max_success_len"]]


def test_library_rollout_counts_dense_grid(C):
    cfg = C.CurationConfig(n_max=32, n_min=4)
    ns = np.arange(0, 1001, dtype=np.int64)
    nt = np.full(1001, 1000, dtype=np.int64)
    got = C.rollout_counts(cfg, ns, nt)
    assert got.tolist() == [CO.rollout_count(k, 1000, n_max=32, n_min=4) for k in range(1001)]


@pytest.mark.parametrize("seed", range(8))
def test_library_curate_batch_matches_oracle(C, seed):
    d, n, caps, tasks = _random_round(seed)
    cfg = C.CurationConfig()
    got = C.curate_batch(cfg, tasks, caps, d["pool"], d["pool_draw"])
    ref = CO.curate_batch(tasks, caps, d["pool"], d["pool_draw"])
    assert got.G == ref["G"]
    assert got.traj_group.tolist() == ref["traj_group"]
    assert got.traj_reward.tolist() == [float(np.float32(r)) for r in ref["traj_reward"]]
    assert got.traj_step_off.tolist() == ref["traj_step_off"]
    assert got.step_tok_off.tolist() == ref["step_tok_off"]
    assert got.traj_source.tolist() == ref["traj_source"]


def test_library_curate_batch_no_pool_and_errors(C):
    from paper_2509_23866_b200 import dart
    cfg = C.CurationConfig()
    tasks = [[([4, 4], 0.0)], [([2], 1.0)]]
    got = C.curate_batch(cfg, tasks, [10, 10])
    assert got.G == 2 and got.traj_source.tolist() == [0, 1]
    with pytest.raises(dart.DartError):
        C.curate_batch(cfg, [[([], 1.0)]], [10])                     # a trajectory with no step
    with pytest.raises(dart.DartError):
        C.curate_batch(cfg, tasks, [0, 10])                          # cap < 1
    with pytest.raises(dart.DartError):
        C.curate_batch(cfg, tasks, [10, 10], [[([1], 1.0)], []], [1.0, 0.0])   # draw outside [0, 1)
    with pytest.raises(dart.DartError):
        C.rollout_counts(cfg, [3], [2])                               # n_success > n_total
    with pytest.raises(dart.DartError):
        C.rollout_counts(C.CurationConfig(n_min=9), [0], [1])         # n_min > n_max


# ------------------------------------------------------------------ the loss pass on a curated batch
@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 1])
def test_loss_pass_on_curated_batch_vs_oracle(C, seed):
    import torch
    from paper_2509_23866_b200 import dart
    from tests.gpu_helpers import compare, run_gpu
    d = synth.make_curation_inputs(10, seed=seed, tok_lo=2, tok_hi=12, max_len=14)
    cfg_c = C.CurationConfig()
    n = C.rollout_counts(cfg_c, d["n_success"], d["n_total"])
    caps = C.trajectory_caps(cfg_c, d["max_success_len"])
    tasks = [d["make_rollouts"](int(n[g]), d["p_succ"][g]) for g in range(10)]
    cb = C.curate_batch(cfg_c, tasks, caps, d["pool"], d["pool_draw"])
    layout = synth.layout_from_csr(cb.G, cb.traj_group, cb.traj_reward, cb.traj_step_off, cb.step_tok_off, seed)
    b = synth.make_batch("curated", seed=seed, layout=layout, V=2000, dtype=torch.bfloat16)
    cfg = dart.Config()
    dl = run_gpu(b, cfg)
    dl.check_status()
    compare(dl, b, cfg)
