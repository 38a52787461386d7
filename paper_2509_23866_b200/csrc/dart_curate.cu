// dart_curate.cu -- SURVEY §8(f) #4 (second half): host-side data curation
// that shapes a DART training batch before the loss pass (§4.1-4.2).
//
// Host code only (no kernels): the trainer's batch builder runs these per
// training iteration on the CPU and hands the resulting CSR metadata
// (dart_meta) to the GPU pass.  Three rules, in the paper's order:
//   * dynamic rollout frequency   PAPER.md:204-206  -> dart_rollout_counts
//   * dynamic trajectory length   PAPER.md:209-211  -> dart_trajectory_caps
//   * experience-pool injection   PAPER.md:214-218  -> dart_curate_batch
// Readings where the paper is silent (DESIGN.md §3 R15-R19) are the ones the
// header states.  Deterministic: random draws are inputs.
#include <cmath>
#include <cstdint>

#include "dart_loss.h"

namespace {

bool cfg_ok(const dart_curation_cfg* c) {
  return c && c->n_min >= 1 && c->n_max >= c->n_min && c->cap_min >= 1 && c->cap_max >= c->cap_min &&
         c->sr_high_permille >= 0 && c->sr_high_permille < 1000;
}

bool set_ok(const dart_traj_set* s) {
  if (!s || s->n_groups < 0) return false;
  if (s->n_groups == 0) return true;
  if (!s->group_off || s->group_off[0] != 0) return false;
  for (int64_t g = 0; g < s->n_groups; ++g)
    if (s->group_off[g + 1] < s->group_off[g]) return false;
  const int64_t n = s->group_off[s->n_groups];
  if (n == 0) return true;
  if (!s->traj_step_off || !s->step_tokens || !s->reward || s->traj_step_off[0] != 0) return false;
  for (int64_t i = 0; i < n; ++i)
    if (s->traj_step_off[i + 1] <= s->traj_step_off[i]) return false;     // >= 1 step per trajectory
  for (int64_t k = 0; k < s->traj_step_off[n]; ++k)
    if (s->step_tokens[k] < 1) return false;                              // >= 1 token per step
  return true;
}

}  // namespace

extern "C" {

dart_status dart_rollout_counts(const dart_curation_cfg* c, int64_t G, const int64_t* n_success,
                                const int64_t* n_total, int32_t* n_rollouts) {
  if (!cfg_ok(c) || G < 0 || (G > 0 && (!n_success || !n_total || !n_rollouts))) return DART_ERR_INVALID_ARG;
  for (int64_t g = 0; g < G; ++g) {
    // counts up to 2^40 keep the exact integer rule below inside int64
    if (n_total[g] < 0 || n_success[g] < 0 || n_success[g] > n_total[g] || n_total[g] > ((int64_t)1 << 40))
      return DART_ERR_INVALID_ARG;
    // exact: sr > h  <=>  1000 ns > h nt ;  drop = floor((1000 ns - h nt) D / ((1000 - h) nt) + 1/2)
    const int64_t ns = n_success[g], nt = n_total[g], h = c->sr_high_permille, D = c->n_max - c->n_min;
    int32_t n = c->n_max;
    if (nt > 0 && 1000 * ns > h * nt) {
      const int64_t num = 2 * (1000 * ns - h * nt) * D + (1000 - h) * nt;
      const int64_t den = 2 * (1000 - h) * nt;
      n = c->n_max - (int32_t)(num / den);      // num, den > 0: integer division = floor
    }
    n_rollouts[g] = n;
  }
  return DART_OK;
}

dart_status dart_trajectory_caps(const dart_curation_cfg* c, int64_t G, const int32_t* max_success_len,
                                 int32_t* caps) {
  if (!cfg_ok(c) || G < 0 || (G > 0 && (!max_success_len || !caps))) return DART_ERR_INVALID_ARG;
  for (int64_t g = 0; g < G; ++g) {
    const int32_t L = max_success_len[g];
    caps[g] = L < 0 ? c->cap_max : (L < c->cap_min ? c->cap_min : (L > c->cap_max ? c->cap_max : L));
  }
  return DART_OK;
}

dart_status dart_curate_batch(const dart_curation_cfg* c, const dart_traj_set* roll, const int32_t* caps,
                              const dart_traj_set* pool, const double* pool_draw, dart_curated* out) {
  if (!cfg_ok(c) || !set_ok(roll) || !caps || !out) return DART_ERR_INVALID_ARG;
  const int64_t G = roll->n_groups;
  const bool has_pool = pool && pool->n_groups > 0;
  if (has_pool && (pool->n_groups != G || !set_ok(pool) || !pool_draw)) return DART_ERR_INVALID_ARG;
  if (!out->traj_group || !out->traj_reward || !out->traj_step_off || !out->step_tok_off || !out->traj_source)
    return DART_ERR_INVALID_ARG;
  for (int64_t g = 0; g < G; ++g)
    if (caps[g] < 1) return DART_ERR_INVALID_ARG;

  int64_t G_out = 0, N = 0, S = 0;
  out->traj_step_off[0] = 0;
  out->step_tok_off[0] = 0;
  // append trajectory i of set s (its first `steps` steps) to the batch
  auto emit = [&](const dart_traj_set* s, int64_t i, int64_t steps, float reward, int64_t source) -> bool {
    if (N + 1 > out->cap_traj || S + steps > out->cap_steps) return false;
    const int64_t k0 = s->traj_step_off[i];
    for (int64_t k = 0; k < steps; ++k) {
      out->step_tok_off[S + 1] = out->step_tok_off[S] + s->step_tokens[k0 + k];
      ++S;
    }
    out->traj_group[N] = (int32_t)G_out;
    out->traj_reward[N] = reward;
    out->traj_source[N] = source;
    out->traj_step_off[N + 1] = S;
    ++N;
    return true;
  };

  for (int64_t g = 0; g < G; ++g) {
    const int64_t r0 = roll->group_off[g], r1 = roll->group_off[g + 1];
    bool any_success = false;
    for (int64_t i = r0; i < r1; ++i) {
      int64_t steps = roll->traj_step_off[i + 1] - roll->traj_step_off[i];
      float reward = roll->reward[i];
      if (steps > caps[g]) {      // terminated at the task's cap before completing: reward 0 (R18)
        steps = caps[g];
        reward = 0.0f;
      }
      if ((double)reward >= c->success_reward) any_success = true;
      if (!emit(roll, i, steps, reward, i)) return DART_ERR_INVALID_ARG;
    }
    if (has_pool && !any_success) {
      const int64_t p0 = pool->group_off[g], p1 = pool->group_off[g + 1];
      if (p1 > p0) {              // every rollout failed: one stored success from the pool (R19)
        const double d = pool_draw[g];
        if (!(d >= 0.0 && d < 1.0)) return DART_ERR_INVALID_ARG;
        int64_t k = (int64_t)std::floor(d * (double)(p1 - p0));
        if (k > p1 - p0 - 1) k = p1 - p0 - 1;
        const int64_t i = p0 + k;
        if (!emit(pool, i, pool->traj_step_off[i + 1] - pool->traj_step_off[i], pool->reward[i], -(i + 1)))
          return DART_ERR_INVALID_ARG;
      }
    }
    if (N > 0 && out->traj_group[N - 1] == (int32_t)G_out) ++G_out;   // this task contributed a group
  }
  out->G = G_out;
  out->N_traj = N;
  out->S = S;
  out->T = out->step_tok_off[S];
  return DART_OK;
}

}  // extern "C"
