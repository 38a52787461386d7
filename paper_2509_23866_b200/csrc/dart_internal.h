// dart_internal.h -- kernel parameter blocks and launchers (internal, C++).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace dart {

// Sweep configuration (compile-time; see DESIGN.md §6 for the sizing).
#ifndef DART_FWD_WARPS
#define DART_FWD_WARPS 8
#endif
#ifndef DART_FWD_STAGES
#define DART_FWD_STAGES 3
#endif
#ifndef DART_BWD_WARPS
#define DART_BWD_WARPS 8
#endif
#ifndef DART_BWD_STAGES
#define DART_BWD_STAGES 4
#endif
constexpr int FWD_WARPS = DART_FWD_WARPS;
constexpr int FWD_STAGES = DART_FWD_STAGES;
constexpr int BWD_WARPS = DART_BWD_WARPS;
constexpr int BWD_STAGES = DART_BWD_STAGES;
// bwd sweep bulk-copy chunk (bytes); the fwd / fused / KL sweeps use CH_BYTES
#ifndef DART_BWD_CHB
#define DART_BWD_CHB 4096
#endif
constexpr int BCH_BYTES = DART_BWD_CHB;
constexpr int BCH_VEC = BCH_BYTES / 16;
// fwd sweep bulk-copy chunk (bytes); canonical segments align to it
#ifndef DART_FWD_CHB
#define DART_FWD_CHB 4096
#endif
constexpr int FCH_BYTES = DART_FWD_CHB;
constexpr int FCH_VEC = FCH_BYTES / 16;

struct AdvParams {
  int64_t G, N_traj, S, T;
  const int32_t* traj_group;
  const float* traj_reward;
  const int64_t* traj_step_off;
  const int64_t* step_tok_off;
  double adv_eps;
  float* adv;
  uint8_t* group_ok;
  int64_t* grp_traj;  // [G+1]
  uint32_t* status;
};

struct TokMetaParams {
  int64_t S, N_traj, T_loc, tok_begin, step_begin, S_loc;
  const int64_t* traj_step_off;
  const int64_t* step_tok_off;
  const float* adv;
  float* tok_adv;
  int32_t* tok_step;
  uint32_t* status;
};

struct FwdParams {
  const uint8_t* logits;
  int64_t ld_bytes, V, T_loc, nvec;
  float c2;  // inv_temperature * log2(e), fp32 (the value every logit is scaled by)
  const int32_t* target;
  const float* logp_old;
  const float* logp_roll;
  const float* logp_ref;
  const float* tok_adv;
  double eps_low, eps_high, is_cap, beta;
  float *lse, *logp, *H, *ell, *dell, *lse2, *aux_w, *aux_kl;
  uint8_t* aux_flags;
  uint32_t* status;
  int lg_nsplit;  // rows are split over 2^lg_nsplit warps (small T_loc)
  // exact-KL mode (dart_kl.cu)
  const uint8_t* ref_logits;
  int64_t ld_ref_bytes;
  float* klq;     // [T_loc] Q_t = ln2 (lse2 - lse2_ref) + KL_t
  float* part_m;
  double *part_s, *part_u;
  uint32_t* row_cnt;
};

struct StepReduceParams {
  int64_t T_loc, tok_begin, step_begin, S_loc;
  const int64_t* step_tok_off;
  const float *H, *aux_kl, *tok_adv;
  float *ell, *dell, *aux_w;       // rewritten per token in step-ratio mode
  uint8_t* aux_flags;
  float* step_entropy;
  double* step_ell;
  double* step_stats;
  // fused mode (dart_loss_fused): no entropy; steps with keep == 0 are skipped
  int no_entropy;
  const uint8_t* keep;  // [S] global, only read when no_entropy
  // step-level ratio (DART_RATIO_STEP)
  int ratio_level;
  int exact_kl;         // DART_KL_EXACT: the KL gradient is per element, not through logp
  const float *logp, *logp_old, *logp_roll, *logp_ref;
  double eps_low, eps_high, is_cap, beta;
  uint32_t* status;     // DART_STATUS_NONFINITE_LOSS of the step-level terms
};

struct SelectParams {
  int64_t G, N_traj, S, T;
  const int64_t* traj_step_off;
  const int64_t* step_tok_off;
  const int64_t* grp_traj;
  const uint8_t* group_ok;
  const float* H;  // [S] global step entropies
  float q;
  int rule;
  uint8_t* keep;
  float* tau;
  int64_t *grp_keep_step, *grp_keep_tok;
};

struct NormParams {
  int64_t G, S, T;
  int norm_mode;
  const int64_t *grp_keep_step, *grp_keep_tok;
  void* norm;  // dart_norm*
};

struct UnpackParams {
  const float* gathered;
  const int64_t* rank_step_off;
  int world;
  int64_t S_pad, S;
  float* H;
};

struct BwdPrepParams {
  int64_t T_loc, tok_begin, step_begin, S_loc, nch;  // nch = chunks per row
  int norm_mode, zero_fill, ratio_level;
  int kept_cost;         // cost units of a kept chunk: 2 (read + write), 3 with exact KL (two reads)
  const int64_t* step_tok_off;
  const uint8_t* keep;   // [S] global
  const void* norm;      // dart_norm*
  const double* step_ell;
  const double* step_stats;
  double* step_scale;    // [S_loc]
  int64_t* step_cost;    // [S_loc+1] prefix of chunk costs (kept 2, masked 1 or 0)
  int64_t* step_chunk;   // [S_loc+1] prefix of chunks that need work
  void* stats;           // dart_stats*
  int no_stats;          // 1: step_scale / step_cost / step_chunk only (step sums not yet written)
  int accumulate;        // 1: add the loss / statistics to *stats instead of overwriting (cfg.stats_accumulate)
};

struct RowRecParams {
  int64_t T_loc, V, ld_bytes;
  int is_bf16;
  const uint8_t* logits;
  const int32_t* tok_step;
  const int32_t* target;
  const double* step_scale;
  const float* dell;
  const float* lse2;
  double invT;
  void* rec;  // int4 [T_loc]: {g, -lse2, y, z_y}  (exact KL: 2 x float4)
  // exact-KL mode
  const uint8_t* ref_logits;
  int64_t ld_ref_bytes;
  const float* klq;
  double beta;
};

struct BwdParams {
  const uint8_t* logits;
  int64_t ld_bytes, V, T_loc, nvec, nch;
  uint8_t* dlogits;
  int64_t ldg_bytes;
  float c2;
  const void* rec;              // int4 [T_loc] row records (K4a)
  const int64_t* step_tok_off;  // global CSR
  int64_t tok_begin, step_begin, S_loc;
  const uint8_t* keep;          // [S] global
  const int64_t* step_cost;     // [S_loc+1] prefix of chunk costs
  const int64_t* step_chunk;    // [S_loc+1] prefix of chunk counts
  int zero_fill;
  // exact-KL mode
  const uint8_t* ref_logits;
  int64_t ld_ref_bytes;
  float invT_f;
};

struct FusedParams {
  const uint8_t* logits;
  int64_t ld_bytes, V, T_loc, nvec, nch;
  int is_bf16, zero_fill;
  uint8_t* dlogits;
  int64_t ldg_bytes;
  float c2;
  double invT, eps_low, eps_high, is_cap, beta;
  const int32_t* target;
  const float *logp_old, *logp_roll, *logp_ref, *tok_adv;
  const int32_t* tok_step;
  const double* step_scale;
  const uint8_t* keep;          // [S] global
  const int64_t* step_cost;     // [S_loc+1]
  const int64_t* step_tok_off;  // global CSR
  int64_t tok_begin, step_begin, S_loc;
  float *lse, *logp, *ell, *dell, *aux_w, *aux_kl;
  uint8_t* aux_flags;
  uint32_t* status;
  void* rec;                    // [T_loc] 32-byte row records (fused_rec_kernel)
};

// LM-head-fused forward (dart_lmhead.cu)
constexpr int LM_NT_PER_CHUNK = 8;   // 256-column tiles per work item (one (m, s, u) partial per row)
constexpr int LM_GROUP_NC = 4;       // vocabulary chunks per raster super-column (L2 reuse of W and h)

struct LmParams {
  int64_t T_loc, V;
  int K;                    // hidden size d
  int n_mb, n_nt, n_nc;     // 128-row blocks, 256-column tiles, vocabulary chunks
  int nt_per_chunk, group_nc;
  int64_t n_items;          // n_mb * n_nc
  float c2;                 // inv_temperature * log2(e)
  const int32_t* target;
  float* part_m;            // [T_loc * n_nc]
  double *part_s, *part_u;  // [T_loc * n_nc]
  float* zy;                // [T_loc] fp32 target logit
  // backward (dz epilogue) mode: non-NULL DZ_n_kept selects it
  const int64_t* DZ_n_kept;   // device count of gathered rows (the A operand's valid rows)
  const void* DZ_rec;         // int4 [n_kept] {g, -lse2, y, local row}
  uint8_t* DZ_out;            // bf16 dz rows [n_kept, ldg]
  int DZ_st256;               // DZ_out and its row pitch 32-byte aligned: 256-bit stores
  int64_t DZ_ldg_bytes;
};

struct LmGatherParams {
  int64_t T_loc, V, d, ld_h, ld_hk, tok_begin, step_begin, S_loc;
  const int32_t* tok_step;
  const int64_t* step_tok_off;
  const uint8_t* keep;        // [S] global
  const int64_t* kept_off;    // [S_loc + 1] exclusive prefix of kept tokens per local step
  const double* step_scale;
  const float* dell;
  const float* lse2;
  const int32_t* target;
  double invT;
  const uint8_t* hidden;      // bf16 [T_loc, ld_h]
  uint8_t* hidden_kept;       // bf16 [>= n_kept, ld_hk]
  void* rec;                  // int4 [T_loc]
  int32_t* kept_rows;         // [T_loc]
  int64_t* n_kept;            // device scalar
};

struct LmCombineParams {
  int n_nc;
  const float* part_m;
  const double *part_s, *part_u;
  const float* zy;
};

cudaError_t launch_lmhead(const void* hidden, int64_t ld_h, const void* weight, int64_t ld_w, const LmParams& p,
                          int num_sms, cudaStream_t st);
cudaError_t launch_lmhead_gather(const LmGatherParams& p, cudaStream_t st);
cudaError_t launch_lmhead_combine(const FwdParams& p, const LmCombineParams& c, cudaStream_t st);

cudaError_t launch_fused_rec(const FusedParams& p, cudaStream_t st);
cudaError_t launch_fwd_kl(const FwdParams& p, bool bf16, int num_sms, cudaStream_t st);
cudaError_t launch_rowrec_kl(const RowRecParams& p, cudaStream_t st);
cudaError_t launch_bwd_kl(const BwdParams& p, bool in_bf16, bool out_bf16, int num_sms, cudaStream_t st);
cudaError_t launch_fused_sweep(const FusedParams& p, bool in_bf16, bool out_bf16, int num_sms, bool split_rows,
                               cudaStream_t st);
cudaError_t launch_adv(const AdvParams& p, cudaStream_t st);
cudaError_t launch_tok_meta(const TokMetaParams& p, cudaStream_t st);
cudaError_t launch_fwd_sweep(const FwdParams& p, bool bf16, int num_sms, cudaStream_t st);
cudaError_t launch_step_reduce(const StepReduceParams& p, cudaStream_t st);
cudaError_t launch_unpack(const UnpackParams& p, cudaStream_t st);
cudaError_t launch_select(const SelectParams& p, cudaStream_t st);
cudaError_t launch_norm(const NormParams& p, cudaStream_t st);
cudaError_t launch_bwd_prep(const BwdPrepParams& p, cudaStream_t st);
cudaError_t launch_rowrec(const RowRecParams& p, cudaStream_t st);
cudaError_t launch_bwd_sweep(const BwdParams& p, bool in_bf16, bool out_bf16, int num_sms, cudaStream_t st);

}  // namespace dart
