"""DART data-curation oracle (§4.1-4.2): plain Python, TEST INFRASTRUCTURE ONLY.

What it computes
----------------
The host-side curation rules that shape a DART training batch before the
policy-loss pass runs on it (the "host-side curation
metadata ... that generates the ragged batches"):

* dynamic rollout frequency  (§4.1 "Dynamic Rollout Frequency")
* dynamic trajectory length  (§4.1 "Dynamic Trajectory Length")
* experience-pool injection  (§4.2 "Experience Pool of Trajectories")

and the CSR batch layout the C ABI takes (include/dart_loss.h dart_meta).
Readings taken where the paper is silent are DESIGN.md §3 R15-R19 and are
repeated at each function.

Who may use it
--------------
Only `tests/` imports this module.  The product implementation is
`dart_rollout_counts` / `dart_trajectory_caps` / `dart_curate_batch` in the
CUDA library's host code (csrc/dart_curate.cu); the two share no code and
neither imports the other.

Everything is written as plain loops over tasks and trajectories, in the
paper's order; the rollout-count rule in exact rational arithmetic
(fractions.Fraction), the pool draw in float64.  Pinned by
tests/test_curation.py against the paper's stated values (8 rollouts at low
success, fewer above 0.6; caps between 10 and 50 steps; at least one positive
trajectory per task after injection), brute-force invariants and hand cases.
"""
from __future__ import annotations

import math
from fractions import Fraction

# Paper constants and readings:
N_MAX = 8            # "reduce its rollout frequency from 8 to lower values"
SR_HIGH = Fraction(3, 5)   # "high success rates (above 0.6)"
N_MIN = 2            # R15: the paper gives no floor; 2 keeps sigma_R computable
CAP_MIN = 10         # "simple clicking tasks might terminate after 10 steps"
CAP_MAX = 50         # "complex multi-application tasks can extend to 50 steps"
SUCCESS_REWARD = 0.5  # R17: reward in [0, 1]; success iff R >= 0.5


def rollout_count(n_success, n_total, n_max=N_MAX, n_min=N_MIN, sr_high=SR_HIGH):
    """PAPER.md:204-206 (§4.1 Dynamic Rollout Frequency): a task keeps the
    maximum sampling n_max while its success rate is at most sr_high; above it
    the rollout count falls (R15: linearly in the success rate, reaching n_min
    at success rate 1, rounded half up to an integer).  No history
    (n_total == 0) counts as success rate 0 ("low success ... maximum sampling").
    Exact rational arithmetic (fractions.Fraction)."""
    sr = Fraction(0) if n_total <= 0 else Fraction(n_success, n_total)
    sr_high = Fraction(sr_high)
    if sr <= sr_high:
        return n_max
    frac = min((sr - sr_high) / (1 - sr_high), Fraction(1))
    drop = math.floor(frac * (n_max - n_min) + Fraction(1, 2))
    return n_max - drop


def trajectory_cap(max_success_len, cap_min=CAP_MIN, cap_max=CAP_MAX):
    """PAPER.md:209-211 (§4.1 Dynamic Trajectory Length): the task's length
    limit is derived from the historical maximum length of its successful
    completions (R16: that maximum, clamped to [cap_min, cap_max]); a task with
    no successful completion yet keeps cap_max ("allowing sufficient
    exploration")."""
    if max_success_len is None or max_success_len < 0:
        return cap_max
    return min(max(max_success_len, cap_min), cap_max)


def is_success(reward, success_reward=SUCCESS_REWARD):
    """R17: a trajectory succeeds iff its reward (in [0, 1]) is >= success_reward."""
    return reward >= success_reward


def curate_batch(tasks, caps, pool, pool_draw, success_reward=SUCCESS_REWARD):
    """Assemble one training batch from per-task rollouts.

    tasks:     list over tasks g of lists of rollouts; a rollout is
               (step_tokens: list of per-step token counts, reward: float).
    caps:      list over tasks of the trajectory cap (trajectory_cap()).
    pool:      list over tasks of lists of pool trajectories (same form);
               every pool trajectory is a stored success.
    pool_draw: list over tasks of a uniform draw in [0, 1) (the random number
               the method uses to pick a pool trajectory; passed in).

    Steps, in the paper's order:
    1. Cap (R18): a rollout longer than its task's cap is
       terminated at the cap; the cut-off trajectory did not complete, so its
       reward becomes 0.
    2. Pool injection (R19): if every (capped) rollout of a
       task fails and the task's pool is not empty, the pool trajectory with
       index floor(draw * len(pool)) is appended to the task's group.
    3. Layout: the task groups in task order, each task's trajectories
       contiguous (rollouts in order, then the injected one), as the CSR
       arrays of dart_meta, plus each trajectory's source (rollout index
       r >= 0 within the flattened rollout list, or -(p + 1) for pool
       trajectory p within the flattened pool list).
    A task with no trajectory at all contributes nothing (no empty groups).
    """
    traj_group, traj_reward, traj_steps, traj_source, step_tokens = [], [], [], [], []
    g_out = 0
    r_flat = 0
    p_base = 0
    for g, rollouts in enumerate(tasks):
        group = []
        for steps, reward in rollouts:
            cap = caps[g]
            if len(steps) > cap:                       # 1. terminated at the cap: not completed
                steps, reward = steps[:cap], 0.0
            group.append((list(steps), float(reward), r_flat))
            r_flat += 1
        if pool[g] and all(not is_success(rw, success_reward) for _, rw, _ in group):
            k = int(math.floor(pool_draw[g] * len(pool[g])))    # 2. draw one stored success
            k = min(k, len(pool[g]) - 1)
            steps, reward = pool[g][k]
            group.append((list(steps), float(reward), -(p_base + k + 1)))
        p_base += len(pool[g])
        if not group:
            continue
        for steps, reward, src in group:                          # 3. layout
            traj_group.append(g_out)
            traj_reward.append(reward)
            traj_steps.append(len(steps))
            traj_source.append(src)
            step_tokens.extend(steps)
        g_out += 1
    traj_step_off = [0]
    for n in traj_steps:
        traj_step_off.append(traj_step_off[-1] + n)
    step_tok_off = [0]
    for n in step_tokens:
        step_tok_off.append(step_tok_off[-1] + n)
    return dict(G=g_out, traj_group=traj_group, traj_reward=traj_reward, traj_step_off=traj_step_off,
                step_tok_off=step_tok_off, traj_source=traj_source)
