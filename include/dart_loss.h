/*
 * dart_loss.h -- C ABI of the B200-native DART policy-loss pass.
 *
 * DART (arXiv 2509.23866), trainer hot path: for every token row of the
 * policy's output logits, a fused log-softmax gives the target log-prob and
 * the entropy (Eq. 1 pi_theta(a|h,s); PAPER.md:238 H_{t,i});
 * step entropies are averaged and the high-entropy steps of
 * each task's step group kept; advantages are
 * group-normalised over the step group D; the
 * token-level truncated IS weight min(pi_old^Train / pi_old^Rollout, C)
 * multiplies the clipped surrogate (Eq. 1,
 * PAPER.md:252-264 Eq. 2) and the optional k3 KL term; the pass returns the
 * loss L = -J_HE (to minimise) and dL/dlogits in bf16 (or fp32).
 *
 * Readings where the paper is silent/ambiguous: DESIGN.md §3.
 *
 * One pass = three calls on the same stream and the same workspace:
 *     dart_loss_fwd      (advantages, fused sweep over all local rows,
 *                         per-step entropy / loss sums)
 *     [caller: all-gather the per-rank step entropies; a no-op at 1 rank]
 *     dart_select_steps  (per-group order-statistic threshold, keep mask,
 *                         global normaliser; identical on every rank)
 *     dart_loss_bwd      (local loss partial + statistics, gradient sweep:
 *                         kept rows read+write, masked rows write zeros)
 *     [caller: all-reduce(SUM) the dart_stats partials]
 *
 * Conventions (all entry points):
 *  - Pointers in the structs are DEVICE pointers unless marked "host".  The
 *    structs themselves are host memory, read during the call only.
 *  - Ownership: the caller allocates every buffer, including the workspace
 *    (size from dart_workspace_size).  The library never allocates, frees,
 *    retains a pointer past the call, or synchronises; every call is
 *    asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream).
 *  - Errors: host-checkable problems return synchronously WITHOUT launching
 *    (DART_ERR_INVALID_ARG / DART_ERR_UNSUPPORTED / DART_ERR_WORKSPACE);
 *    a failed launch returns DART_ERR_CUDA.  Data errors found on the device
 *    OR bits into *status (DART_STATUS_* below); the caller checks it after
 *    the stream synchronises.  Outputs are unspecified when a bit is set.
 *  - Determinism: bitwise deterministic for fixed inputs and device; no
 *    floating-point atomics.  Per-row reductions use a canonical order that
 *    does not depend on how rows are distributed, so sharding a batch over
 *    ranks reproduces the single-rank bits (tests/test_virtual_ranks.py).
 *  - Layout: logits row t (local) starts at logits + t*ld elements; rows must
 *    be 16-byte aligned (base 16 B aligned, ld*sizeof(elem) % 16 == 0).
 */
#ifndef DART_LOSS_H
#define DART_LOSS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DART_ABI_VERSION 6

typedef enum {
  DART_OK = 0,
  DART_ERR_INVALID_ARG = 1,   /* NULL / misaligned pointer, bad size or config value */
  DART_ERR_UNSUPPORTED = 2,   /* dtype or mode not supported */
  DART_ERR_CUDA = 3,          /* kernel launch / CUDA runtime failure */
  DART_ERR_WORKSPACE = 4      /* ws_bytes < dart_workspace_size(...) or ws NULL */
} dart_status;

typedef enum { DART_BF16 = 0, DART_F32 = 1 } dart_dtype;

/* Normalisation of E over D (token aggregation unstated). */
typedef enum {
  DART_NORM_TOKEN_MEAN_KEPT = 0, /* L = sum_{kept tokens} ell / N_keep_tok   (default, DAPO-style) */
  DART_NORM_STEP_MEAN_KEPT = 1,  /* L = (1/N_keep_step) sum_{kept s} (1/n_s) sum_{t in s} ell */
  DART_NORM_TOKEN_MEAN_ALL = 2,  /* L = sum_{kept tokens} ell / T_global */
  DART_NORM_STEP_MEAN_ALL = 3,   /* L = (1/S_global) sum_{kept s} (1/n_s) sum_{t in s} ell */
  DART_NORM_SUM = 4              /* L = sum_{kept tokens} ell */
} dart_norm_mode;

/* Threshold tau_g over the n_g ascending-sorted step entropies s[] of group g
 * ("at least larger than 20% steps", 264 tau_D^{0.2}). */
typedef enum {
  DART_SEL_FLOOR = 0,  /* tau = s[floor(q*n)]            (default; keeps >= ceil((1-q)n)) */
  DART_SEL_CEIL = 1,   /* tau = s[min(ceil(q*n), n-1)] */
  DART_SEL_LINEAR = 2, /* tau = s[lo] + f*(s[lo+1]-s[lo]), pos = q*(n-1)  (torch.quantile) */
  DART_SEL_OFF = 3     /* keep every step of a valid group */
} dart_select_rule;
/* q*n and q*(n-1) are evaluated in float64 from the float32 value of entropy_q. */

/* Granularity of the importance ratio r = pi_theta / pi_old^Train and of the
 * truncated IS weight. */
typedef enum {
  DART_RATIO_TOKEN = 0,  /* per token: r_t = exp(logp_t - logp_old_t), w_t = min(exp(logp_old_t - logp_roll_t), C);
                            ell_t = -w_t min(r_t A, clip(r_t) A) + beta k3_t                  (default) */
  DART_RATIO_STEP = 1    /* per step (the literal pi(a|h,s) of Eq. 1/2): r_s = exp(sum_{t in s} logp_t - logp_old_t),
                            w_s = min(exp(sum_t logp_old_t - logp_roll_t), C);
                            ell_s = -w_s min(r_s A, clip(r_s) A) + beta sum_{t in s} k3_t, and
                            L = sum_{kept s} inv_norm * ell_s (no 1/n_s factor in any mode);
                            out.ell[t] holds ell_s / n_s and step_ell[s] holds ell_s */
} dart_ratio_level;

/* KL(pi_theta || pi_ref) estimator for the beta term (
 * the estimator is unstated -- SURVEY Q10, §8(f) NEXT #4). */
typedef enum {
  DART_KL_K3 = 0,    /* per-token k3 from log pi_ref(y_t): e^d - d - 1, d = logp_ref - logp (default) */
  DART_KL_EXACT = 1  /* exact full-vocabulary KL_t = sum_v p_v (log p_v - log q_v) from the reference
                        policy's logits (batch->ref_logits, same temperature); its gradient
                        invT p_v ((log p_v - log q_v) - KL_t) enters every element of the row */
} dart_kl_mode;

/* Device status bits (OR-accumulated into *status). */
#define DART_STATUS_NONFINITE_LOGIT (1u << 0) /* NaN or +inf logit in a row */
#define DART_STATUS_TARGET_RANGE    (1u << 1) /* target outside [0, V) */
#define DART_STATUS_ROW_ALL_NEGINF  (1u << 2) /* every logit of a row is -inf */
#define DART_STATUS_NONFINITE_LOGP  (1u << 3) /* non-finite logp_old / logp_rollout / logp_ref */
#define DART_STATUS_EMPTY           (1u << 4) /* a step with 0 tokens or a trajectory with 0 steps */
#define DART_STATUS_BAD_CSR         (1u << 5) /* decreasing offsets, traj_group decreasing or out of
                                                 [0,G), or the local shard not aligned to steps */
#define DART_STATUS_TARGET_NEGINF   (1u << 6) /* the target's logit is -inf (log-prob -inf) */
#define DART_STATUS_NONFINITE_LOSS  (1u << 7) /* a token's loss term or its derivative is not finite in
                                                 the fp32 outputs (ell / dell), e.g. the k3 term
                                                 e^d - d - 1 at d = logp_ref - logp > 88.7 or an
                                                 importance ratio exp(logp - logp_old) beyond fp32 */

/* Hyper-parameters (host struct).  Paper values: PAPER.md:575-578. */
typedef struct {
  float eps_low;          /* 0.2   clip lower bound 1-eps_low,  in (0,1)            */
  float eps_high;         /* 0.28  clip upper bound 1+eps_high, in (0,1)            */
  float is_cap;           /* C = 1 truncation of the IS weight, > 0                 */
  float beta_kl;          /* 0.1   k3-KL coefficient, >= 0; 0 => logp_ref may be NULL */
  float entropy_q;        /* 0.2   drop quantile, in [0,1)                           */
  float inv_temperature;  /* 1.0   logits are scaled by this before the softmax, (0, 1e6] */
  float adv_eps;          /* 0.0 (paper).  > 0: A = (R-mean)/(std+adv_eps) and sigma=0
                             groups are kept with A = 0 (a verl-style flag)          */
  int32_t norm_mode;      /* dart_norm_mode   */
  int32_t select_rule;    /* dart_select_rule */
  int32_t zero_fill_masked; /* 1: dense dlogits (masked rows written as zeros);
                               0: masked rows are left untouched                   */
  int32_t ratio_level;    /* dart_ratio_level */
  int32_t kl_mode;        /* dart_kl_mode */
  int32_t stats_accumulate; /* 0: dart_loss_bwd / dart_loss_fused / dart_lmhead_bwd overwrite *stats;
                               1: they ADD this call's loss and statistics to *stats (fixed-order fp64
                               adds in stream order: deterministic) -- a batch streamed as chunks
                               (virtual ranks) then totals its statistics inside the library */
} dart_cfg;

/* GLOBAL batch metadata, replicated on every rank (device pointers). */
typedef struct {
  int64_t G;        /* task groups (step groups D) */
  int64_t N_traj;   /* trajectories */
  int64_t S;        /* steps */
  int64_t T;        /* tokens = step_tok_off[S] */
  const int32_t* traj_group;     /* [N_traj] group id in [0,G), non-decreasing */
  const float* traj_reward;      /* [N_traj] R_i (in [0,1]) */
  const int64_t* traj_step_off;  /* [N_traj+1] steps of traj i: [off[i], off[i+1]), >= 1 each */
  const int64_t* step_tok_off;   /* [S+1] global tokens of step s, >= 1 each */
} dart_meta;

/* The LOCAL shard: a contiguous range of whole trajectories. */
typedef struct {
  const void* logits;      /* [T_loc, ld] elements of logits_dtype */
  int32_t logits_dtype;    /* dart_dtype */
  int64_t T_loc;           /* local token rows (>= 0) */
  int64_t V;               /* vocabulary size (>= 1) */
  int64_t ld;              /* row pitch in elements, >= V */
  int64_t tok_begin;       /* global token index of local row 0 (= step_tok_off[step_begin]) */
  int64_t step_begin;      /* global step index of local step 0 */
  int64_t S_loc;           /* local steps */
  const int32_t* target;       /* [T_loc] sampled token y_t in [0,V) */
  const float* logp_old;       /* [T_loc] log pi_old^Train(y_t)   (stop-grad input) */
  const float* logp_rollout;   /* [T_loc] log pi_old^Rollout(y_t) (recorded by the rollout engine) */
  const float* logp_ref;       /* [T_loc] log pi_ref(y_t), or NULL when beta_kl == 0 or kl_mode == EXACT */
  const void* ref_logits;      /* [T_loc, ld_ref] reference-policy logits (logits_dtype), only read when
                                  kl_mode == DART_KL_EXACT and beta_kl > 0; 16-byte aligned rows */
  int64_t ld_ref;              /* row pitch of ref_logits in elements, >= V */
} dart_batch;

/* Forward outputs (caller-allocated device buffers). */
typedef struct {
  float* lse;           /* [T_loc] log-sum-exp of z*inv_temperature (natural log) */
  float* logp;          /* [T_loc] log pi_theta(y_t) */
  float* tok_entropy;   /* [T_loc] H_t (nats) */
  float* ell;           /* [T_loc] per-token loss term -w*min(rA, clip(r)A) + beta*k3 */
  float* dell;          /* [T_loc] d ell / d logp */
  float* step_entropy;  /* [S_loc] mean token entropy of each local step */
  double* step_ell;     /* [S_loc] sum of ell over each local step's tokens */
  float* adv;           /* [N_traj] advantage per trajectory (global) */
  uint8_t* group_ok;    /* [G] 1 iff sigma_R > 0 (or adv_eps > 0) */
  uint32_t* status;     /* [1] DART_STATUS_* bits, OR-accumulated (caller zeroes it) */
} dart_fwd_out;

/* Normaliser, written by dart_select_steps (device struct). */
typedef struct {
  int64_t n_keep_tok;   /* global kept tokens */
  int64_t n_keep_step;  /* global kept steps */
  int64_t n_tok;        /* global tokens T */
  int64_t n_step;       /* global steps S */
  double inv_norm;      /* 1/N for the mode (0 if N == 0); per-step 1/n_s applied in bwd */
} dart_norm;

/* Local partial sums, written by dart_loss_bwd (device struct).  All-reduce
 * (SUM) over ranks; loss is already normalised (sum over ranks = L). */
typedef struct {
  double loss;
  double n_tok;        /* local tokens */
  double n_kept_tok;   /* local kept tokens */
  double n_kept_step;  /* local kept steps */
  double sum_clip;     /* kept tokens whose clipped branch is the min (no ratio gradient) */
  double sum_trunc;    /* kept tokens with pi_old/pi_rollout >= C */
  double sum_w;        /* sum of IS weights over kept tokens */
  double sum_adv;      /* sum of A over kept tokens */
  double sum_adv2;     /* sum of A^2 over kept tokens */
  double sum_H;        /* sum of token entropies over all local tokens */
  double sum_kl;       /* sum of k3 KL over kept tokens */
} dart_stats;

/* Bytes of workspace the three calls need for this shard (host-only, no launch). */
size_t dart_workspace_size(const dart_batch* batch, const dart_meta* meta, const dart_cfg* cfg);

/* Forward: advantages (all G groups), metadata checks, the fused sweep over
 * all T_loc rows (one read of each logit row), per-step reductions.
 * `out` fields are all required.  Workspace contents carry to select/bwd. */
dart_status dart_loss_fwd(const dart_batch* batch, const dart_meta* meta, const dart_cfg* cfg,
                          const dart_fwd_out* out, void* workspace, size_t ws_bytes, void* stream);

/* Selection over the GLOBAL step entropies.
 * step_entropy_gathered: [world * S_pad] floats, rank r's S_loc_r step
 *   entropies at [r*S_pad, r*S_pad + S_loc_r) (the layout of an all-gather of
 *   per-rank buffers padded to S_pad); for world == 1 pass the fwd's
 *   step_entropy with S_pad = S.
 * rank_step_off: [world+1] device int64, rank r owns global steps
 *   [rank_step_off[r], rank_step_off[r+1]); rank_step_off[world] == S.
 * Writes keep [S] (uint8), tau [G] (float; NaN for empty groups) and *norm. */
dart_status dart_select_steps(const float* step_entropy_gathered, const int64_t* rank_step_off,
                              int32_t world, int64_t S_pad, const dart_meta* meta,
                              const dart_cfg* cfg, const uint8_t* group_ok, uint8_t* keep,
                              float* tau, dart_norm* norm, void* workspace, size_t ws_bytes,
                              void* stream);

/* Backward: local loss partial + statistics into *stats, then dL/dlogits for
 * the local rows: kept rows re-read once and written once, masked rows
 * written as zeros (zero_fill_masked=1) or skipped.  dlogits: [T_loc, ldg]
 * of grad_dtype, 16-byte aligned rows.
 * dlogits == NULL: loss-only mode -- *stats (loss, counts, sums) without the
 * gradient sweep; batch->logits / logits_dtype / ld / ref_logits and
 * grad_dtype / ldg are then ignored (e.g. after dart_lmhead_fwd). */
dart_status dart_loss_bwd(const dart_batch* batch, const dart_meta* meta, const dart_cfg* cfg,
                          const dart_fwd_out* fwd, const uint8_t* keep, const dart_norm* norm,
                          void* dlogits, int32_t grad_dtype, int64_t ldg, dart_stats* stats,
                          void* workspace, size_t ws_bytes, void* stream);

/* single-read fused loss + gradient when the step
 * mask is known in advance: `keep` / `norm` come from dart_loss_fwd +
 * dart_select_steps run on the old-policy pass (whose logp is this call's
 * logp_old; at the first update theta = theta_old, so its entropies are the
 * paper's).  Each kept row is read from HBM once (its second,
 * gradient pass hits L2) and its gradient written once; masked rows are
 * written as zeros (zero_fill_masked) without being read.  Token-level
 * ratio only (DART_ERR_UNSUPPORTED for DART_RATIO_STEP).  Writes out->lse,
 * logp, ell, dell for rows of kept steps (masked rows' per-token outputs are
 * left untouched), out->step_ell, out->adv, out->group_ok, out->status,
 * *stats (sum_H = 0: no entropies are computed) and dlogits. */
dart_status dart_loss_fused(const dart_batch* batch, const dart_meta* meta, const dart_cfg* cfg,
                            const uint8_t* keep, const dart_norm* norm, const dart_fwd_out* out,
                            void* dlogits, int32_t grad_dtype, int64_t ldg, dart_stats* stats,
                            void* workspace, size_t ws_bytes, void* stream);

/* the LM-head operand of dart_lmhead_fwd.  The
 * policy logits are z_{t,v} = sum_k h_{t,k} W_{v,k} (the softmax of z / T is
 * pi_theta(a|h,s), Eq. 1); they are computed on the tensor cores
 * tile by tile and reduced in the epilogue, never written to memory.
 * Both operands bf16, K (= d) contiguous, 16-byte aligned base, row pitch in
 * elements with pitch*2 % 16 == 0, d % 8 == 0. */
typedef struct {
  const void* hidden;   /* [T_loc, ld_h] bf16: last hidden state of the local token rows */
  const void* weight;   /* [V, ld_w] bf16: LM-head weight (the nn.Linear [out, in] layout) */
  int64_t d;            /* hidden size (K of the contraction), >= 8 */
  int64_t ld_h;         /* row pitch of hidden, >= d */
  int64_t ld_w;         /* row pitch of weight, >= d */
} dart_lmhead;

/* Workspace for dart_lmhead_fwd (>= dart_workspace_size(batch, ...); the
 * same buffer then serves dart_select_steps). */
size_t dart_lmhead_workspace_size(const dart_lmhead* head, const dart_batch* batch, const dart_meta* meta,
                                  const dart_cfg* cfg);

/* Forward of the loss pass with the LM head fused in: identical outputs to
 * dart_loss_fwd on the logits z = h W^T (fp32 accumulation on the tensor
 * cores, no rounding to bf16), without the [T_loc, V] logits ever existing.
 * batch->logits / logits_dtype / ld are ignored (may be NULL/0); V, the
 * targets, logp_old/rollout/ref and the shard fields are used as in
 * dart_loss_fwd.  Use: the theta_old "old log-prob" pass that produces the
 * token entropies, step entropies and (via dart_select_steps) the step mask
 * for dart_loss_fused.  DART_ERR_UNSUPPORTED for kl_mode == DART_KL_EXACT
 * with beta_kl > 0.  The backward through the head: dart_lmhead_bwd. */
dart_status dart_lmhead_fwd(const dart_lmhead* head, const dart_batch* batch, const dart_meta* meta,
                            const dart_cfg* cfg, const dart_fwd_out* out, void* workspace, size_t ws_bytes,
                            void* stream);

/* SURVEY §8(f) NEXT #3, training half -- the loss gradient through the LM
 * head with the logits still never in memory.  Call after dart_lmhead_fwd on
 * the same head, shard, workspace and `fwd` outputs (the update pass's own
 * forward at theta; at theta = theta_old it is the old-log-prob pass itself),
 * with the step mask / normaliser (keep, norm) of dart_select_steps.
 *   1. *stats: local loss partial and statistics (as dart_loss_bwd).
 *   2. The KEPT rows of the shard (rows of masked steps have no gradient,
 *      PAPER.md:256 indicator) are gathered in row order: kept_rows[i] = the
 *      local row of compact row i, *n_kept = their count K (device scalar),
 *      hidden_kept row i = hidden row kept_rows[i].
 *   3. z = hidden_kept W^T is recomputed on the tensor cores tile by tile
 *      (tcgen05, TMEM accumulators) and the epilogue writes
 *        dz[i, v] = g_t (delta_{v, y_t} - exp(z_{t,v} invT - lse_t)),
 *        g_t = c_s dell_t invT          (SURVEY Q11 c_s),
 *      rounded to bf16 (RNE): dz = dL/dz of the kept rows.
 * The model's backward through the head is then two plain GEMMs the caller
 * runs (e.g. cuBLAS): dL/dh[kept_rows] = dz W, dL/dW = dz^T hidden_kept; all
 * other rows of dL/dh are zero.
 * Buffers (device, caller-owned, sized for T_loc rows since K is known on the
 * device only): dz [T_loc, ldg] bf16 with ldg >= V, ldg % 8 == 0;
 * hidden_kept [T_loc, ld_hk] bf16 with ld_hk >= d, ld_hk % 8 == 0; kept_rows
 * int32 [T_loc]; n_kept int64 [1]; all 16-byte aligned.  Rows >= K of dz /
 * hidden_kept / kept_rows are left untouched.  Workspace: the
 * dart_lmhead_workspace_size buffer of the forward (its per-row state is
 * read).  Same errors as dart_lmhead_fwd. */
dart_status dart_lmhead_bwd(const dart_lmhead* head, const dart_batch* batch, const dart_meta* meta,
                            const dart_cfg* cfg, const dart_fwd_out* fwd, const uint8_t* keep,
                            const dart_norm* norm, void* dz, int64_t ldg, void* hidden_kept, int64_t ld_hk,
                            int32_t* kept_rows, int64_t* n_kept, dart_stats* stats, void* workspace,
                            size_t ws_bytes, void* stream);

/* Single-rank convenience: fwd + select (world = 1) + bwd on one stream. */
dart_status dart_loss_pass(const dart_batch* batch, const dart_meta* meta, const dart_cfg* cfg,
                           const dart_fwd_out* fwd, uint8_t* keep, float* tau, dart_norm* norm,
                           void* dlogits, int32_t grad_dtype, int64_t ldg, dart_stats* stats,
                           void* workspace, size_t ws_bytes, void* stream);

/* Static description of a status code (never NULL). */
const char* dart_status_str(dart_status s);

/* ABI version (DART_ABI_VERSION) -- lets bindings check they match. */
int32_t dart_abi_version(void);

/* Number of kernel launches the most recent successful fwd / select / bwd
 * call on this host thread issued (for the bench's gpu_launches count). */
int32_t dart_last_launch_count(void);

/* Profiling hook (host thread-local): when set, the next fwd / bwd calls
 * record these cudaEvent_t handles on their stream immediately before and
 * after the sweep kernel (K1 resp. K4), so the caller can time the hot
 * kernels alone with CUDA events.  Pass NULLs to disable.  Events are owned
 * by the caller. */
void dart_set_timing_events(void* fwd_sweep_begin, void* fwd_sweep_end, void* bwd_sweep_begin,
                            void* bwd_sweep_end);

/* ==================================================================
 * SURVEY §8(f) #4 (second half) -- host-side data curation (PAPER.md
 * §4.1-4.2): the per-iteration rules that shape the ragged batch whose
 * CSR metadata (dart_meta) the loss pass above consumes.  HOST functions
 * (host pointers, no stream, no GPU), deterministic: the one random draw
 * the method makes (which pool trajectory to inject) is an input.
 * Readings where the paper is silent: DESIGN.md §3 R15-R19.
 * ================================================================== */
typedef struct {
  int32_t n_max;          /* rollouts per task at low success rate: 8 */
  int32_t n_min;          /* rollouts at success rate 1 (R15, paper silent): 2 */
  int32_t cap_min;        /* shortest trajectory cap: 10 steps */
  int32_t cap_max;        /* longest trajectory cap: 50 steps */
  int32_t sr_high_permille; /* success rate above which sampling is reduced, in 1/1000: 600;
                               integer so the rule is exact rational arithmetic (no float ties) */
  int32_t reserved;       /* 0 */
  double success_reward;  /* R17: a trajectory succeeds iff reward >= this: 0.5 (rewards in [0,1]) */
} dart_curation_cfg;

/* Trajectories grouped by task, as CSR (host pointers, caller-owned):
 * task g owns trajectories [group_off[g], group_off[g+1]); trajectory i owns
 * steps [traj_step_off[i], traj_step_off[i+1]) (>= 1 step), step k has
 * step_tokens[k] >= 1 tokens; reward[i] in [0, 1]. */
typedef struct {
  int64_t n_groups;
  const int64_t* group_off;       /* [n_groups + 1], group_off[0] == 0, non-decreasing */
  const int64_t* traj_step_off;   /* [N + 1], strictly increasing from 0 */
  const int32_t* step_tokens;     /* [S] */
  const float* reward;            /* [N] */
} dart_traj_set;

/* Output of dart_curate_batch (host buffers, caller-owned, capacities in
 * cap_traj / cap_steps): the dart_meta CSR of the batch plus each
 * trajectory's source (rollout index i >= 0, or -(p + 1) for pool
 * trajectory p).  G, N_traj, S, T are written by the call. */
typedef struct {
  int64_t cap_traj, cap_steps;    /* in: capacities of the arrays below */
  int32_t* traj_group;            /* [cap_traj]      task group (0..G-1, non-decreasing) */
  float* traj_reward;             /* [cap_traj]      R_i */
  int64_t* traj_source;           /* [cap_traj]      provenance */
  int64_t* traj_step_off;         /* [cap_traj + 1]  CSR steps */
  int64_t* step_tok_off;          /* [cap_steps + 1] CSR tokens */
  int64_t G, N_traj, S, T;        /* out: sizes */
} dart_curated;

/* PAPER.md:204-206 (§4.1 Dynamic Rollout Frequency): rollouts to sample for
 * each of G tasks from its success history (n_success of n_total past
 * rollouts; n_total == 0 counts as success rate 0).  sr <= sr_high -> n_max;
 * above, linearly down to n_min at sr = 1, rounded half up (R15):
 *   n = n_max - floor((sr - sr_high) / (1 - sr_high) * (n_max - n_min) + 1/2)
 * evaluated exactly in integers (sr = n_success / n_total, sr_high =
 * sr_high_permille / 1000).  DART_ERR_INVALID_ARG on a bad config or counts
 * (negative, n_success > n_total, or n_total > 2^40). */
dart_status dart_rollout_counts(const dart_curation_cfg* cfg, int64_t G, const int64_t* n_success,
                                const int64_t* n_total, int32_t* n_rollouts);

/* PAPER.md:209-211 (§4.1 Dynamic Trajectory Length): each task's step cap
 * from the historical maximum length of its successful completions
 * (max_success_len[g] < 0: none yet -> cap_max), clamped to
 * [cap_min, cap_max] (R16). */
dart_status dart_trajectory_caps(const dart_curation_cfg* cfg, int64_t G, const int32_t* max_success_len,
                                 int32_t* caps);

/* PAPER.md:209-218 (§4.1-4.2): one training batch from this iteration's
 * rollouts.  Per task, in order: (1) a rollout longer than the task's cap is
 * terminated at the cap and, not having completed, gets reward 0 (R18);
 * (2) if every rollout of the task then fails and the task's pool is not
 * empty, pool trajectory floor(pool_draw[g] * n_pool_g) (a stored success,
 * PAPER.md:216) is appended to the group (R19); (3) the task's trajectories
 * (rollouts in order, then the injected one) form one contiguous group; a
 * task with no trajectory forms none.  pool may be NULL (no pool) or must
 * have n_groups == rollouts->n_groups; pool_draw[g] in [0, 1).
 * DART_ERR_INVALID_ARG on malformed CSR, bad caps / draws or too small
 * output capacities (cap_traj >= N_rollouts + G and cap_steps >= steps of
 * all rollouts + pool suffice). */
dart_status dart_curate_batch(const dart_curation_cfg* cfg, const dart_traj_set* rollouts, const int32_t* caps,
                              const dart_traj_set* pool, const double* pool_draw, dart_curated* out);

#ifdef __cplusplus
}
#endif
#endif /* DART_LOSS_H */
