// dart_abi.cu -- the C ABI of include/dart_loss.h: host-side argument
// validation, the workspace layout, and the kernel launch sequence.
// Never allocates, never synchronises; every launch goes to `stream`.
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <nvtx3/nvToolsExt.h>

#include "dart_common.cuh"
#include "dart_internal.h"

using namespace dart;

namespace {

// NVTX range over one ABI call (header-only NVTX3: a no-op unless a profiler
// such as nsys / ncu --nvtx injects itself), so timelines show the phases.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

thread_local int32_t g_launches = 0;
thread_local int32_t g_last_launches = 0;
thread_local cudaEvent_t g_ev[4] = {nullptr, nullptr, nullptr, nullptr};

void rec(int i, cudaStream_t s) {
  if (g_ev[i]) (void)cudaEventRecord(g_ev[i], s);
}

int sm_count() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  static int cache[64] = {0};
  if (dev >= 0 && dev < 64 && cache[dev]) return cache[dev];
  int n = 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  if (dev >= 0 && dev < 64) cache[dev] = n;
  return n;
}

inline size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline size_t esize(int32_t dt) { return dt == DART_BF16 ? 2 : 4; }

// Global-metadata regions first (their offsets depend only on S and G, so
// dart_select_steps can address them without knowing the shard), then the
// per-shard regions.
size_t ws_global_prefix(const dart_meta* m, WsLayout* L) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += al256(bytes ? bytes : 1);
    return o;
  };
  const size_t S = (size_t)(m->S > 0 ? m->S : 0);
  const size_t G = (size_t)(m->G > 0 ? m->G : 0);
  const size_t h = take(S * 4), gt = take((G + 1) * 8), gs = take(G * 8), gk = take(G * 8);
  if (L) {
    L->H_glob = h;
    L->grp_traj = gt;
    L->grp_keep_step = gs;
    L->grp_keep_tok = gk;
  }
  return off;
}

WsLayout ws_layout(const dart_batch* b, const dart_meta* m) {
  WsLayout L;
  size_t off = ws_global_prefix(m, &L);
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += al256(bytes ? bytes : 1);
    return o;
  };
  const size_t T = (size_t)(b->T_loc > 0 ? b->T_loc : 0);
  const size_t S_loc = (size_t)(b->S_loc > 0 ? b->S_loc : 0);
  L.tok_adv = take(T * 4);
  L.tok_step = take(T * 4);
  L.lse2 = take(T * 4);
  L.aux_w = take(T * 4);
  L.aux_kl = take(T * 4);
  L.aux_flags = take(T);
  L.rec = take(T * 32);
  L.klq = take(T * 4);
  L.step_stats = take(S_loc * NSTAT * 8);
  L.step_cost = take((S_loc + 1) * 8);
  L.step_scale = take(S_loc * 8);
  L.step_chunk = take((S_loc + 1) * 8);
  L.split_alloc = T > 0 && T <= (size_t)SPLIT_MAX_ROWS;
  if (L.split_alloc) {
    L.part_m = take(T * KSEG * 4);
    L.part_s = take(T * KSEG * 8);
    L.part_u = take(T * KSEG * 8);
    L.row_cnt = take(T * 4);
  } else {
    L.part_m = L.part_s = L.part_u = L.row_cnt = 0;
  }
  L.fused_rec = take(T * 32);
  L.bwd_misc = take(256);
  L.total = off;
  return L;
}

template <typename T>
inline T* at(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<uint8_t*>(ws) + off);
}

bool cfg_ok(const dart_cfg* c) {
  if (!c) return false;
  if (!(c->eps_low > 0.f && c->eps_low < 1.f)) return false;
  if (!(c->eps_high > 0.f && c->eps_high < 1.f)) return false;
  if (!(c->is_cap > 0.f) || !std::isfinite(c->is_cap)) return false;
  if (!(c->beta_kl >= 0.f) || !std::isfinite(c->beta_kl)) return false;
  if (!(c->entropy_q >= 0.f && c->entropy_q < 1.f)) return false;
  if (!(c->inv_temperature > 0.f && c->inv_temperature <= 1e6f)) return false;
  if (!(c->adv_eps >= 0.f) || !std::isfinite(c->adv_eps)) return false;
  if (c->norm_mode < DART_NORM_TOKEN_MEAN_KEPT || c->norm_mode > DART_NORM_SUM) return false;
  if (c->select_rule < DART_SEL_FLOOR || c->select_rule > DART_SEL_OFF) return false;
  if (c->ratio_level != DART_RATIO_TOKEN && c->ratio_level != DART_RATIO_STEP) return false;
  if (c->kl_mode != DART_KL_K3 && c->kl_mode != DART_KL_EXACT) return false;
  if (c->stats_accumulate != 0 && c->stats_accumulate != 1) return false;
  return true;
}

bool meta_ok(const dart_meta* m) {
  if (!m) return false;
  if (m->G < 0 || m->N_traj < 0 || m->S < 0 || m->T < 0) return false;
  if (m->N_traj > 0 && m->G < 1) return false;
  if (!m->traj_step_off || !m->step_tok_off) return false;
  if (m->N_traj > 0 && (!m->traj_group || !m->traj_reward)) return false;
  if (m->T > ((int64_t)1 << 40)) return false;
  return true;
}

// need_logits = false: the logits fields are ignored (LM-head forward, loss-only bwd)
dart_status batch_check(const dart_batch* b, const dart_meta* m, const dart_cfg* c, bool need_logits = true) {
  if (!b || !meta_ok(m) || !cfg_ok(c)) return DART_ERR_INVALID_ARG;
  if (need_logits && b->logits_dtype != DART_BF16 && b->logits_dtype != DART_F32) return DART_ERR_UNSUPPORTED;
  if (b->T_loc < 0 || b->V < 1 || (need_logits && b->ld < b->V) || b->S_loc < 0) return DART_ERR_INVALID_ARG;
  if (b->V > 0x7fffffffLL) return DART_ERR_INVALID_ARG;
  if (b->tok_begin < 0 || b->tok_begin + b->T_loc > m->T) return DART_ERR_INVALID_ARG;
  if (b->step_begin < 0 || b->step_begin + b->S_loc > m->S) return DART_ERR_INVALID_ARG;
  if (b->T_loc > 0) {
    if ((need_logits && !b->logits) || !b->target || !b->logp_old || !b->logp_rollout) return DART_ERR_INVALID_ARG;
    if (c->beta_kl > 0.f && c->kl_mode == DART_KL_K3 && !b->logp_ref) return DART_ERR_INVALID_ARG;
    if (need_logits && c->beta_kl > 0.f && c->kl_mode == DART_KL_EXACT) {
      if (!b->ref_logits || !aligned16(b->ref_logits) || b->ld_ref < b->V ||
          ((size_t)b->ld_ref * esize(b->logits_dtype)) % 16 != 0)
        return DART_ERR_INVALID_ARG;
    }
    if (need_logits && (!aligned16(b->logits) || ((size_t)b->ld * esize(b->logits_dtype)) % 16 != 0))
      return DART_ERR_INVALID_ARG;
    if (b->S_loc < 1) return DART_ERR_INVALID_ARG;
  }
  return DART_OK;
}

dart_status fwd_out_check(const dart_batch* b, const dart_meta* m, const dart_fwd_out* o) {
  if (!o || !o->status) return DART_ERR_INVALID_ARG;
  if (b->T_loc > 0 && (!o->lse || !o->logp || !o->tok_entropy || !o->ell || !o->dell)) return DART_ERR_INVALID_ARG;
  if (b->S_loc > 0 && (!o->step_entropy || !o->step_ell)) return DART_ERR_INVALID_ARG;
  if (m->N_traj > 0 && !o->adv) return DART_ERR_INVALID_ARG;
  if (m->G > 0 && !o->group_ok) return DART_ERR_INVALID_ARG;
  return DART_OK;
}

dart_status cuda_status(cudaError_t e) {
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return DART_ERR_CUDA;
  }
  ++g_launches;
  return DART_OK;
}

// log2 of the number of warps a row is split over: only for few rows, and
// only when every canonical segment is non-empty (rows >= KSEG chunks)
inline bool exact_kl(const dart_cfg* c) { return c->kl_mode == DART_KL_EXACT && c->beta_kl > 0.f; }

int choose_lg_nsplit(const dart_batch* b, const WsLayout& L, int64_t nvec) {
  if (!L.split_alloc || nvec < (int64_t)KSEG * FCH_VEC) return 0;
  const int64_t target_units = 4LL * sm_count() * 16;
  int lg = 0;
  while ((1 << lg) < KSEG && (b->T_loc << lg) < target_units) ++lg;
  return lg;
}

// LM-head workspace tail and argument checks
struct LmLayout {
  int n_mb, n_nt, n_nc;
  size_t part_m, part_s, part_u, zy, total;
};

LmLayout lm_layout(const dart_batch* b, const dart_meta* m) {
  LmLayout L;
  const int64_t T = b->T_loc > 0 ? b->T_loc : 0;
  L.n_mb = (int)((T + 127) / 128);
  L.n_nt = (int)((b->V + 255) / 256);
  L.n_nc = (L.n_nt + LM_NT_PER_CHUNK - 1) / LM_NT_PER_CHUNK;
  size_t off = ws_layout(b, m).total;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += al256(bytes ? bytes : 1);
    return o;
  };
  L.part_m = take((size_t)T * L.n_nc * 4);
  L.part_s = take((size_t)T * L.n_nc * 8);
  L.part_u = take((size_t)T * L.n_nc * 8);
  L.zy = take((size_t)T * 4);
  L.total = off;
  return L;
}

dart_status lmhead_check(const dart_lmhead* h, const dart_batch* b, const dart_meta* m, const dart_cfg* c) {
  if (!h || !b) return DART_ERR_INVALID_ARG;
  if (c && cfg_ok(c) && exact_kl(c)) return DART_ERR_UNSUPPORTED;   // needs the reference logits
  dart_status st = batch_check(b, m, c, /*need_logits=*/false);
  if (st != DART_OK) return st;
  if (h->d < 8 || h->d % 8 != 0 || h->d > (1 << 20)) return DART_ERR_INVALID_ARG;
  if (h->ld_h < h->d || h->ld_w < h->d || h->ld_h % 8 != 0 || h->ld_w % 8 != 0) return DART_ERR_INVALID_ARG;
  if (b->T_loc > 0 && (!h->hidden || !h->weight || !aligned16(h->hidden) || !aligned16(h->weight)))
    return DART_ERR_INVALID_ARG;
  if (b->T_loc >= ((int64_t)1 << 31)) return DART_ERR_INVALID_ARG;
  return DART_OK;
}
}  // namespace

#define DART_TRY(expr)                        \
  do {                                        \
    dart_status _s = cuda_status((expr));     \
    if (_s != DART_OK) return _s;             \
  } while (0)
// runtime calls that are not kernels of ours (not counted as launches)
#define DART_TRY_RT(expr)                     \
  do {                                        \
    if ((expr) != cudaSuccess) {              \
      (void)cudaGetLastError();               \
      return DART_ERR_CUDA;                   \
    }                                         \
  } while (0)

extern "C" {

int32_t dart_abi_version(void) { return DART_ABI_VERSION; }

int32_t dart_last_launch_count(void) { return g_last_launches; }

void dart_set_timing_events(void* a, void* b, void* c, void* d) {
  g_ev[0] = static_cast<cudaEvent_t>(a);
  g_ev[1] = static_cast<cudaEvent_t>(b);
  g_ev[2] = static_cast<cudaEvent_t>(c);
  g_ev[3] = static_cast<cudaEvent_t>(d);
}

const char* dart_status_str(dart_status s) {
  switch (s) {
    case DART_OK: return "DART_OK";
    case DART_ERR_INVALID_ARG: return "DART_ERR_INVALID_ARG: invalid argument (NULL/misaligned pointer, size or config value)";
    case DART_ERR_UNSUPPORTED: return "DART_ERR_UNSUPPORTED: unsupported dtype or mode";
    case DART_ERR_CUDA: return "DART_ERR_CUDA: CUDA launch or runtime failure";
    case DART_ERR_WORKSPACE: return "DART_ERR_WORKSPACE: workspace missing or smaller than dart_workspace_size()";
  }
  return "DART_UNKNOWN_STATUS";
}

size_t dart_workspace_size(const dart_batch* b, const dart_meta* m, const dart_cfg* c) {
  (void)c;
  if (!b || !m) return 0;
  return ws_layout(b, m).total;
}

dart_status dart_loss_fwd(const dart_batch* b, const dart_meta* m, const dart_cfg* c, const dart_fwd_out* o,
                          void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("dart_loss_fwd");
  dart_status st = batch_check(b, m, c);
  if (st != DART_OK) return st;
  if ((st = fwd_out_check(b, m, o)) != DART_OK) return st;
  const WsLayout L = ws_layout(b, m);
  if (!ws || ws_bytes < L.total) return DART_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  g_launches = 0;

  // K0a: advantages of all G groups + metadata checks
  AdvParams ap;
  ap.G = m->G; ap.N_traj = m->N_traj; ap.S = m->S; ap.T = m->T;
  ap.traj_group = m->traj_group; ap.traj_reward = m->traj_reward;
  ap.traj_step_off = m->traj_step_off; ap.step_tok_off = m->step_tok_off;
  ap.adv_eps = (double)c->adv_eps;
  ap.adv = o->adv; ap.group_ok = o->group_ok;
  ap.grp_traj = at<int64_t>(ws, L.grp_traj);
  ap.status = o->status;
  DART_TRY(launch_adv(ap, s));

  // K0b: token -> (step, A) tables
  TokMetaParams tp;
  tp.S = m->S; tp.N_traj = m->N_traj; tp.T_loc = b->T_loc; tp.tok_begin = b->tok_begin;
  tp.step_begin = b->step_begin; tp.S_loc = b->S_loc;
  tp.traj_step_off = m->traj_step_off; tp.step_tok_off = m->step_tok_off;
  tp.adv = o->adv;
  tp.tok_adv = at<float>(ws, L.tok_adv);
  tp.tok_step = at<int32_t>(ws, L.tok_step);
  tp.status = o->status;
  DART_TRY(launch_tok_meta(tp, s));

  if (b->T_loc > 0) {
    const size_t es = esize(b->logits_dtype);
    const int64_t nvec = (int64_t)((b->V * es + 15) / 16);
    FwdParams fp;
    fp.logits = static_cast<const uint8_t*>(b->logits);
    fp.ld_bytes = b->ld * (int64_t)es;
    fp.V = b->V; fp.T_loc = b->T_loc; fp.nvec = nvec;
    fp.c2 = (float)((double)c->inv_temperature * LOG2E_D);
    fp.target = b->target; fp.logp_old = b->logp_old; fp.logp_roll = b->logp_rollout;
    fp.logp_ref = b->logp_ref;
    fp.tok_adv = at<float>(ws, L.tok_adv);
    fp.eps_low = c->eps_low; fp.eps_high = c->eps_high; fp.is_cap = c->is_cap; fp.beta = c->beta_kl;
    fp.lse = o->lse; fp.logp = o->logp; fp.H = o->tok_entropy; fp.ell = o->ell; fp.dell = o->dell;
    fp.lse2 = at<float>(ws, L.lse2);
    fp.aux_w = at<float>(ws, L.aux_w);
    fp.aux_kl = at<float>(ws, L.aux_kl);
    fp.aux_flags = at<uint8_t>(ws, L.aux_flags);
    fp.status = o->status;
    fp.lg_nsplit = exact_kl(c) ? 0 : choose_lg_nsplit(b, L, nvec);
    fp.ref_logits = static_cast<const uint8_t*>(b->ref_logits);
    fp.ld_ref_bytes = b->ld_ref * (int64_t)es;
    fp.klq = at<float>(ws, L.klq);
    fp.part_m = L.split_alloc ? at<float>(ws, L.part_m) : nullptr;
    fp.part_s = L.split_alloc ? at<double>(ws, L.part_s) : nullptr;
    fp.part_u = L.split_alloc ? at<double>(ws, L.part_u) : nullptr;
    fp.row_cnt = L.split_alloc ? at<uint32_t>(ws, L.row_cnt) : nullptr;
    if (fp.lg_nsplit > 0) DART_TRY_RT(cudaMemsetAsync(fp.row_cnt, 0, (size_t)b->T_loc * 4, s));
    rec(0, s);
    if (exact_kl(c)) DART_TRY(launch_fwd_kl(fp, b->logits_dtype == DART_BF16, sm_count(), s));
    else DART_TRY(launch_fwd_sweep(fp, b->logits_dtype == DART_BF16, sm_count(), s));
    rec(1, s);

    StepReduceParams sp;
    sp.T_loc = b->T_loc; sp.tok_begin = b->tok_begin; sp.step_begin = b->step_begin; sp.S_loc = b->S_loc;
    sp.step_tok_off = m->step_tok_off;
    sp.H = o->tok_entropy; sp.ell = o->ell; sp.dell = o->dell;
    sp.aux_w = fp.aux_w; sp.aux_kl = fp.aux_kl; sp.tok_adv = fp.tok_adv; sp.aux_flags = fp.aux_flags;
    sp.ratio_level = c->ratio_level;
    sp.exact_kl = exact_kl(c) ? 1 : 0;
    sp.no_entropy = 0;
    sp.keep = nullptr;
    sp.logp = o->logp; sp.logp_old = b->logp_old; sp.logp_roll = b->logp_rollout; sp.logp_ref = b->logp_ref;
    sp.eps_low = c->eps_low; sp.eps_high = c->eps_high; sp.is_cap = c->is_cap; sp.beta = c->beta_kl;
    sp.status = o->status;
    sp.step_entropy = o->step_entropy; sp.step_ell = o->step_ell;
    sp.step_stats = at<double>(ws, L.step_stats);
    DART_TRY(launch_step_reduce(sp, s));
  }
  g_last_launches = g_launches;
  return DART_OK;
}

size_t dart_lmhead_workspace_size(const dart_lmhead* h, const dart_batch* b, const dart_meta* m,
                                  const dart_cfg* c) {
  (void)h;
  (void)c;
  if (!b || !m) return 0;
  return lm_layout(b, m).total;
}

dart_status dart_lmhead_fwd(const dart_lmhead* h, const dart_batch* b, const dart_meta* m, const dart_cfg* c,
                            const dart_fwd_out* o, void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("dart_lmhead_fwd");
  dart_status st = lmhead_check(h, b, m, c);
  if (st != DART_OK) return st;
  if ((st = fwd_out_check(b, m, o)) != DART_OK) return st;
  const WsLayout L = ws_layout(b, m);
  const LmLayout LL = lm_layout(b, m);
  if (!ws || ws_bytes < LL.total) return DART_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  g_launches = 0;

  AdvParams ap;
  ap.G = m->G; ap.N_traj = m->N_traj; ap.S = m->S; ap.T = m->T;
  ap.traj_group = m->traj_group; ap.traj_reward = m->traj_reward;
  ap.traj_step_off = m->traj_step_off; ap.step_tok_off = m->step_tok_off;
  ap.adv_eps = (double)c->adv_eps;
  ap.adv = o->adv; ap.group_ok = o->group_ok;
  ap.grp_traj = at<int64_t>(ws, L.grp_traj);
  ap.status = o->status;
  DART_TRY(launch_adv(ap, s));

  TokMetaParams tp;
  tp.S = m->S; tp.N_traj = m->N_traj; tp.T_loc = b->T_loc; tp.tok_begin = b->tok_begin;
  tp.step_begin = b->step_begin; tp.S_loc = b->S_loc;
  tp.traj_step_off = m->traj_step_off; tp.step_tok_off = m->step_tok_off;
  tp.adv = o->adv;
  tp.tok_adv = at<float>(ws, L.tok_adv);
  tp.tok_step = at<int32_t>(ws, L.tok_step);
  tp.status = o->status;
  DART_TRY(launch_tok_meta(tp, s));

  if (b->T_loc > 0) {
    LmParams lp = {};
    lp.T_loc = b->T_loc; lp.V = b->V; lp.K = (int)h->d;
    lp.n_mb = LL.n_mb; lp.n_nt = LL.n_nt; lp.n_nc = LL.n_nc;
    lp.nt_per_chunk = LM_NT_PER_CHUNK; lp.group_nc = LM_GROUP_NC;
    lp.n_items = (int64_t)LL.n_mb * LL.n_nc;
    lp.c2 = (float)((double)c->inv_temperature * LOG2E_D);
    lp.target = b->target;
    lp.part_m = at<float>(ws, LL.part_m);
    lp.part_s = at<double>(ws, LL.part_s);
    lp.part_u = at<double>(ws, LL.part_u);
    lp.zy = at<float>(ws, LL.zy);
    rec(0, s);
    DART_TRY(launch_lmhead(h->hidden, h->ld_h, h->weight, h->ld_w, lp, sm_count(), s));
    rec(1, s);

    FwdParams fp;
    memset(&fp, 0, sizeof(fp));
    fp.V = b->V; fp.T_loc = b->T_loc;
    fp.c2 = lp.c2;
    fp.target = b->target; fp.logp_old = b->logp_old; fp.logp_roll = b->logp_rollout;
    fp.logp_ref = b->logp_ref;
    fp.tok_adv = at<float>(ws, L.tok_adv);
    fp.eps_low = c->eps_low; fp.eps_high = c->eps_high; fp.is_cap = c->is_cap; fp.beta = c->beta_kl;
    fp.lse = o->lse; fp.logp = o->logp; fp.H = o->tok_entropy; fp.ell = o->ell; fp.dell = o->dell;
    fp.lse2 = at<float>(ws, L.lse2);
    fp.aux_w = at<float>(ws, L.aux_w);
    fp.aux_kl = at<float>(ws, L.aux_kl);
    fp.aux_flags = at<uint8_t>(ws, L.aux_flags);
    fp.status = o->status;
    LmCombineParams cp;
    cp.n_nc = LL.n_nc;
    cp.part_m = lp.part_m; cp.part_s = lp.part_s; cp.part_u = lp.part_u; cp.zy = lp.zy;
    DART_TRY(launch_lmhead_combine(fp, cp, s));

    StepReduceParams sp;
    sp.T_loc = b->T_loc; sp.tok_begin = b->tok_begin; sp.step_begin = b->step_begin; sp.S_loc = b->S_loc;
    sp.step_tok_off = m->step_tok_off;
    sp.H = o->tok_entropy; sp.ell = o->ell; sp.dell = o->dell;
    sp.aux_w = fp.aux_w; sp.aux_kl = fp.aux_kl; sp.tok_adv = fp.tok_adv; sp.aux_flags = fp.aux_flags;
    sp.ratio_level = c->ratio_level;
    sp.exact_kl = 0;
    sp.no_entropy = 0;
    sp.keep = nullptr;
    sp.logp = o->logp; sp.logp_old = b->logp_old; sp.logp_roll = b->logp_rollout; sp.logp_ref = b->logp_ref;
    sp.eps_low = c->eps_low; sp.eps_high = c->eps_high; sp.is_cap = c->is_cap; sp.beta = c->beta_kl;
    sp.status = o->status;
    sp.step_entropy = o->step_entropy; sp.step_ell = o->step_ell;
    sp.step_stats = at<double>(ws, L.step_stats);
    DART_TRY(launch_step_reduce(sp, s));
  }
  g_last_launches = g_launches;
  return DART_OK;
}

dart_status dart_lmhead_bwd(const dart_lmhead* h, const dart_batch* b, const dart_meta* m, const dart_cfg* c,
                            const dart_fwd_out* f, const uint8_t* keep, const dart_norm* norm, void* dz, int64_t ldg,
                            void* hidden_kept, int64_t ld_hk, int32_t* kept_rows, int64_t* n_kept, dart_stats* stats,
                            void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("dart_lmhead_bwd");
  dart_status st = lmhead_check(h, b, m, c);
  if (st != DART_OK) return st;
  if ((st = fwd_out_check(b, m, f)) != DART_OK) return st;
  if (!norm || !stats || !n_kept || (m->S > 0 && !keep)) return DART_ERR_INVALID_ARG;
  if (b->T_loc > 0) {
    if (!dz || !hidden_kept || !kept_rows || !aligned16(dz) || !aligned16(hidden_kept)) return DART_ERR_INVALID_ARG;
    if (ldg < b->V || ldg % 8 != 0 || ld_hk < h->d || ld_hk % 8 != 0) return DART_ERR_INVALID_ARG;
  }
  const WsLayout L = ws_layout(b, m);
  const LmLayout LL = lm_layout(b, m);
  if (!ws || ws_bytes < LL.total) return DART_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  g_launches = 0;

  // K6 with unit costs: step_cost = exclusive prefix of kept tokens per local step
  BwdPrepParams pp = {};
  pp.T_loc = b->T_loc; pp.tok_begin = b->tok_begin; pp.step_begin = b->step_begin; pp.S_loc = b->S_loc;
  pp.nch = 1; pp.norm_mode = c->norm_mode; pp.zero_fill = 0; pp.ratio_level = c->ratio_level;
  pp.kept_cost = 1;
  pp.step_tok_off = m->step_tok_off; pp.keep = keep; pp.norm = norm;
  pp.step_ell = f->step_ell; pp.step_stats = at<double>(ws, L.step_stats);
  pp.step_scale = at<double>(ws, L.step_scale);
  pp.step_cost = at<int64_t>(ws, L.step_cost);
  pp.step_chunk = at<int64_t>(ws, L.step_chunk);
  pp.stats = stats;
  pp.no_stats = 0;
  pp.accumulate = c->stats_accumulate ? 1 : 0;
  DART_TRY(launch_bwd_prep(pp, s));

  LmGatherParams gp;
  gp.T_loc = b->T_loc; gp.V = b->V; gp.d = h->d; gp.ld_h = h->ld_h; gp.ld_hk = ld_hk;
  gp.tok_begin = b->tok_begin; gp.step_begin = b->step_begin; gp.S_loc = b->S_loc;
  gp.tok_step = at<int32_t>(ws, L.tok_step);
  gp.step_tok_off = m->step_tok_off;
  gp.keep = keep;
  gp.kept_off = pp.step_cost;
  gp.step_scale = pp.step_scale;
  gp.dell = f->dell;
  gp.lse2 = at<float>(ws, L.lse2);
  gp.target = b->target;
  gp.invT = (double)c->inv_temperature;
  gp.hidden = static_cast<const uint8_t*>(h->hidden);
  gp.hidden_kept = static_cast<uint8_t*>(hidden_kept);
  gp.rec = at<int4>(ws, L.rec);
  gp.kept_rows = kept_rows;
  gp.n_kept = n_kept;
  DART_TRY(launch_lmhead_gather(gp, s));

  if (b->T_loc > 0) {
    LmParams lp = {};
    lp.T_loc = b->T_loc; lp.V = b->V; lp.K = (int)h->d;
    lp.n_mb = LL.n_mb; lp.n_nt = LL.n_nt; lp.n_nc = LL.n_nc;
    lp.nt_per_chunk = LM_NT_PER_CHUNK; lp.group_nc = LM_GROUP_NC;
    lp.n_items = (int64_t)LL.n_mb * LL.n_nc;
    lp.c2 = (float)((double)c->inv_temperature * LOG2E_D);
    lp.DZ_n_kept = n_kept;
    lp.DZ_rec = gp.rec;
    lp.DZ_out = static_cast<uint8_t*>(dz);
    lp.DZ_ldg_bytes = ldg * 2;
    lp.DZ_st256 = ((reinterpret_cast<uintptr_t>(dz) & 31) == 0 && (lp.DZ_ldg_bytes & 31) == 0) ? 1 : 0;
    rec(2, s);
    DART_TRY(launch_lmhead(hidden_kept, ld_hk, h->weight, h->ld_w, lp, sm_count(), s));
    rec(3, s);
  }
  g_last_launches = g_launches;
  return DART_OK;
}

dart_status dart_select_steps(const float* gathered, const int64_t* rank_step_off, int32_t world, int64_t S_pad,
                              const dart_meta* m, const dart_cfg* c, const uint8_t* group_ok, uint8_t* keep,
                              float* tau, dart_norm* norm, void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("dart_select_steps");
  if (!meta_ok(m) || !cfg_ok(c)) return DART_ERR_INVALID_ARG;
  if (world < 1 || S_pad < 0) return DART_ERR_INVALID_ARG;
  if (!norm || (m->S > 0 && (!gathered || !keep)) || (m->G > 0 && (!group_ok || !tau))) return DART_ERR_INVALID_ARG;
  if (world > 1 && !rank_step_off) return DART_ERR_INVALID_ARG;
  if (world == 1 && S_pad < m->S) return DART_ERR_INVALID_ARG;
  if ((int64_t)world * S_pad < m->S) return DART_ERR_INVALID_ARG;
  WsLayout L;
  const size_t need = ws_global_prefix(m, &L);
  if (!ws || ws_bytes < need) return DART_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  g_launches = 0;

  const float* H = gathered;
  if (world > 1) {  // all-gather layout -> global step order
    UnpackParams up;
    up.gathered = gathered; up.rank_step_off = rank_step_off; up.world = world;
    up.S_pad = S_pad; up.S = m->S;
    up.H = at<float>(ws, L.H_glob);
    DART_TRY(launch_unpack(up, s));
    H = up.H;
  }
  SelectParams sp;
  sp.G = m->G; sp.N_traj = m->N_traj; sp.S = m->S; sp.T = m->T;
  sp.traj_step_off = m->traj_step_off; sp.step_tok_off = m->step_tok_off;
  sp.grp_traj = at<int64_t>(ws, L.grp_traj);
  sp.group_ok = group_ok; sp.H = H;
  sp.q = c->entropy_q; sp.rule = c->select_rule;
  sp.keep = keep; sp.tau = tau;
  sp.grp_keep_step = at<int64_t>(ws, L.grp_keep_step);
  sp.grp_keep_tok = at<int64_t>(ws, L.grp_keep_tok);
  DART_TRY(launch_select(sp, s));

  NormParams np;
  np.G = m->G; np.S = m->S; np.T = m->T; np.norm_mode = c->norm_mode;
  np.grp_keep_step = sp.grp_keep_step; np.grp_keep_tok = sp.grp_keep_tok;
  np.norm = norm;
  DART_TRY(launch_norm(np, s));
  g_last_launches = g_launches;
  return DART_OK;
}

dart_status dart_loss_bwd(const dart_batch* b, const dart_meta* m, const dart_cfg* c, const dart_fwd_out* f,
                          const uint8_t* keep, const dart_norm* norm, void* dlogits, int32_t grad_dtype,
                          int64_t ldg, dart_stats* stats, void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("dart_loss_bwd");
  const bool loss_only = dlogits == nullptr;   // loss + statistics only: no gradient sweep, logits unused
  dart_status st = batch_check(b, m, c, !loss_only);
  if (st != DART_OK) return st;
  if ((st = fwd_out_check(b, m, f)) != DART_OK) return st;
  if (!loss_only && grad_dtype != DART_BF16 && grad_dtype != DART_F32) return DART_ERR_UNSUPPORTED;
  if (!norm || !stats || (m->S > 0 && !keep)) return DART_ERR_INVALID_ARG;
  if (b->T_loc > 0 && !loss_only) {
    if (!dlogits || ldg < b->V || !aligned16(dlogits) || ((size_t)ldg * esize(grad_dtype)) % 16 != 0)
      return DART_ERR_INVALID_ARG;
  }
  const WsLayout L = ws_layout(b, m);
  if (!ws || ws_bytes < L.total) return DART_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  g_launches = 0;
  const size_t es = esize(b->logits_dtype);
  const int64_t nvec = (int64_t)((b->V * es + 15) / 16);
  const bool kx = exact_kl(c);
  const int64_t chv = kx ? CH_VEC / 2 : BCH_VEC;           // exact KL: 2 KB of z + 2 KB of z_ref per slot
  const int64_t nch = (nvec + chv - 1) / chv;

  BwdPrepParams pp = {};
  pp.T_loc = b->T_loc; pp.tok_begin = b->tok_begin; pp.step_begin = b->step_begin; pp.S_loc = b->S_loc;
  pp.nch = nch; pp.norm_mode = c->norm_mode; pp.zero_fill = c->zero_fill_masked ? 1 : 0;
  pp.ratio_level = c->ratio_level;
  pp.kept_cost = kx ? 3 : 2;
  pp.step_tok_off = m->step_tok_off; pp.keep = keep; pp.norm = norm;
  pp.step_ell = f->step_ell; pp.step_stats = at<double>(ws, L.step_stats);
  pp.step_scale = at<double>(ws, L.step_scale);
  pp.step_cost = at<int64_t>(ws, L.step_cost);
  pp.step_chunk = at<int64_t>(ws, L.step_chunk);
  pp.stats = stats;
  pp.no_stats = 0;
  pp.accumulate = c->stats_accumulate ? 1 : 0;
  DART_TRY(launch_bwd_prep(pp, s));

  if (b->T_loc > 0 && !loss_only) {
    RowRecParams rp = {};
    rp.T_loc = b->T_loc; rp.V = b->V; rp.ld_bytes = b->ld * (int64_t)es;
    rp.is_bf16 = b->logits_dtype == DART_BF16;
    rp.logits = static_cast<const uint8_t*>(b->logits);
    rp.tok_step = at<int32_t>(ws, L.tok_step); rp.target = b->target; rp.step_scale = pp.step_scale;
    rp.dell = f->dell; rp.lse2 = at<float>(ws, L.lse2); rp.invT = (double)c->inv_temperature;
    rp.rec = at<int4>(ws, L.rec);
    rp.ref_logits = static_cast<const uint8_t*>(b->ref_logits);
    rp.ld_ref_bytes = b->ld_ref * (int64_t)es;
    rp.klq = at<float>(ws, L.klq);
    rp.beta = c->beta_kl;
    if (kx) DART_TRY(launch_rowrec_kl(rp, s));
    else DART_TRY(launch_rowrec(rp, s));

    BwdParams bp;
    bp.logits = static_cast<const uint8_t*>(b->logits);
    bp.ld_bytes = b->ld * (int64_t)es;
    bp.V = b->V; bp.T_loc = b->T_loc; bp.nvec = nvec; bp.nch = nch;
    bp.dlogits = static_cast<uint8_t*>(dlogits);
    bp.ldg_bytes = ldg * (int64_t)esize(grad_dtype);
    bp.c2 = (float)((double)c->inv_temperature * LOG2E_D);
    bp.rec = rp.rec;
    bp.step_tok_off = m->step_tok_off;
    bp.tok_begin = b->tok_begin; bp.step_begin = b->step_begin; bp.S_loc = b->S_loc;
    bp.keep = keep;
    bp.step_cost = pp.step_cost;
    bp.step_chunk = pp.step_chunk;
    bp.zero_fill = pp.zero_fill;
    bp.ref_logits = rp.ref_logits;
    bp.ld_ref_bytes = rp.ld_ref_bytes;
    bp.invT_f = c->inv_temperature;
    rec(2, s);
    if (kx) DART_TRY(launch_bwd_kl(bp, b->logits_dtype == DART_BF16, grad_dtype == DART_BF16, sm_count(), s));
    else DART_TRY(launch_bwd_sweep(bp, b->logits_dtype == DART_BF16, grad_dtype == DART_BF16, sm_count(), s));
    rec(3, s);
  }
  g_last_launches = g_launches;
  return DART_OK;
}

dart_status dart_loss_fused(const dart_batch* b, const dart_meta* m, const dart_cfg* c, const uint8_t* keep,
                            const dart_norm* norm, const dart_fwd_out* o, void* dlogits, int32_t grad_dtype,
                            int64_t ldg, dart_stats* stats, void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("dart_loss_fused");
  dart_status st = batch_check(b, m, c);
  if (st != DART_OK) return st;
  if (c->ratio_level != DART_RATIO_TOKEN || exact_kl(c)) return DART_ERR_UNSUPPORTED;
  if (!o || !o->status) return DART_ERR_INVALID_ARG;
  if (b->T_loc > 0 && (!o->lse || !o->logp || !o->ell || !o->dell)) return DART_ERR_INVALID_ARG;
  if (b->S_loc > 0 && !o->step_ell) return DART_ERR_INVALID_ARG;
  if ((m->N_traj > 0 && !o->adv) || (m->G > 0 && !o->group_ok)) return DART_ERR_INVALID_ARG;
  if (grad_dtype != DART_BF16 && grad_dtype != DART_F32) return DART_ERR_UNSUPPORTED;
  if (!norm || !stats || (m->S > 0 && !keep)) return DART_ERR_INVALID_ARG;
  if (b->T_loc > 0) {
    if (!dlogits || ldg < b->V || !aligned16(dlogits) || ((size_t)ldg * esize(grad_dtype)) % 16 != 0)
      return DART_ERR_INVALID_ARG;
  }
  const WsLayout L = ws_layout(b, m);
  if (!ws || ws_bytes < L.total) return DART_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  g_launches = 0;
  const size_t es = esize(b->logits_dtype);
  const int64_t nvec = (int64_t)((b->V * es + 15) / 16);
  const int64_t nch = (nvec + CH_VEC - 1) / CH_VEC;

  AdvParams ap;
  ap.G = m->G; ap.N_traj = m->N_traj; ap.S = m->S; ap.T = m->T;
  ap.traj_group = m->traj_group; ap.traj_reward = m->traj_reward;
  ap.traj_step_off = m->traj_step_off; ap.step_tok_off = m->step_tok_off;
  ap.adv_eps = (double)c->adv_eps;
  ap.adv = o->adv; ap.group_ok = o->group_ok;
  ap.grp_traj = at<int64_t>(ws, L.grp_traj);
  ap.status = o->status;
  DART_TRY(launch_adv(ap, s));
  TokMetaParams tp;
  tp.S = m->S; tp.N_traj = m->N_traj; tp.T_loc = b->T_loc; tp.tok_begin = b->tok_begin;
  tp.step_begin = b->step_begin; tp.S_loc = b->S_loc;
  tp.traj_step_off = m->traj_step_off; tp.step_tok_off = m->step_tok_off;
  tp.adv = o->adv;
  tp.tok_adv = at<float>(ws, L.tok_adv);
  tp.tok_step = at<int32_t>(ws, L.tok_step);
  tp.status = o->status;
  DART_TRY(launch_tok_meta(tp, s));

  BwdPrepParams pp = {};   // per-step loss weights + chunk-cost prefix (the mask is known)
  pp.T_loc = b->T_loc; pp.tok_begin = b->tok_begin; pp.step_begin = b->step_begin; pp.S_loc = b->S_loc;
  pp.nch = nch; pp.norm_mode = c->norm_mode; pp.zero_fill = c->zero_fill_masked ? 1 : 0;
  pp.ratio_level = c->ratio_level;
  pp.kept_cost = 2;
  pp.step_tok_off = m->step_tok_off; pp.keep = keep; pp.norm = norm;
  pp.step_ell = o->step_ell; pp.step_stats = at<double>(ws, L.step_stats);
  pp.step_scale = at<double>(ws, L.step_scale);
  pp.step_cost = at<int64_t>(ws, L.step_cost);
  pp.step_chunk = at<int64_t>(ws, L.step_chunk);
  pp.stats = stats;
  pp.no_stats = b->T_loc > 0 ? 1 : 0;   // the step sums come from the sweep below; stats in the second call
  pp.accumulate = c->stats_accumulate ? 1 : 0;
  DART_TRY(launch_bwd_prep(pp, s));

  if (b->T_loc > 0) {
    FusedParams fp = {};
    fp.logits = static_cast<const uint8_t*>(b->logits);
    fp.ld_bytes = b->ld * (int64_t)es;
    fp.V = b->V; fp.T_loc = b->T_loc; fp.nvec = nvec; fp.nch = nch;
    fp.is_bf16 = b->logits_dtype == DART_BF16; fp.zero_fill = pp.zero_fill;
    fp.dlogits = static_cast<uint8_t*>(dlogits);
    fp.ldg_bytes = ldg * (int64_t)esize(grad_dtype);
    fp.c2 = (float)((double)c->inv_temperature * LOG2E_D);
    fp.invT = c->inv_temperature; fp.eps_low = c->eps_low; fp.eps_high = c->eps_high;
    fp.is_cap = c->is_cap; fp.beta = c->beta_kl;
    fp.target = b->target; fp.logp_old = b->logp_old; fp.logp_roll = b->logp_rollout; fp.logp_ref = b->logp_ref;
    fp.tok_adv = tp.tok_adv; fp.tok_step = tp.tok_step; fp.step_scale = pp.step_scale;
    fp.keep = keep; fp.step_cost = pp.step_cost; fp.step_tok_off = m->step_tok_off;
    fp.tok_begin = b->tok_begin; fp.step_begin = b->step_begin; fp.S_loc = b->S_loc;
    fp.lse = o->lse; fp.logp = o->logp; fp.ell = o->ell; fp.dell = o->dell;
    fp.aux_w = at<float>(ws, L.aux_w); fp.aux_kl = at<float>(ws, L.aux_kl);
    fp.aux_flags = at<uint8_t>(ws, L.aux_flags);
    fp.status = o->status;
    fp.rec = at<uint8_t>(ws, L.fused_rec);
    DART_TRY(launch_fused_rec(fp, s));
    rec(2, s);
    // rows split over a 2-CTA cluster (the pass-2 re-read then hits L2); one CTA per
    // row for rows of a single chunk
    DART_TRY(launch_fused_sweep(fp, fp.is_bf16, grad_dtype == DART_BF16, sm_count(), fp.nch >= 2, s));
    rec(3, s);

    StepReduceParams sp;
    sp.T_loc = b->T_loc; sp.tok_begin = b->tok_begin; sp.step_begin = b->step_begin; sp.S_loc = b->S_loc;
    sp.step_tok_off = m->step_tok_off;
    sp.H = nullptr; sp.ell = o->ell; sp.dell = o->dell;
    sp.aux_w = fp.aux_w; sp.aux_kl = fp.aux_kl; sp.tok_adv = fp.tok_adv; sp.aux_flags = fp.aux_flags;
    sp.step_entropy = nullptr; sp.step_ell = o->step_ell;
    sp.step_stats = at<double>(ws, L.step_stats);
    sp.no_entropy = 1; sp.keep = keep; sp.exact_kl = 0;
    sp.ratio_level = DART_RATIO_TOKEN;
    sp.logp = o->logp; sp.logp_old = b->logp_old; sp.logp_roll = b->logp_rollout; sp.logp_ref = b->logp_ref;
    sp.eps_low = c->eps_low; sp.eps_high = c->eps_high; sp.is_cap = c->is_cap; sp.beta = c->beta_kl;
    sp.status = o->status;
    DART_TRY(launch_step_reduce(sp, s));
    pp.no_stats = 0;
    DART_TRY(launch_bwd_prep(pp, s));   // loss partial + statistics from the step sums
  }
  g_last_launches = g_launches;
  return DART_OK;
}

dart_status dart_loss_pass(const dart_batch* b, const dart_meta* m, const dart_cfg* c, const dart_fwd_out* f,
                           uint8_t* keep, float* tau, dart_norm* norm, void* dlogits, int32_t grad_dtype,
                           int64_t ldg, dart_stats* stats, void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("dart_loss_pass");
  dart_status st = batch_check(b, m, c);
  if (st != DART_OK) return st;
  // single rank: the shard must be the whole batch
  if (b->tok_begin != 0 || b->T_loc != m->T || b->step_begin != 0 || b->S_loc != m->S) return DART_ERR_INVALID_ARG;
  int32_t total = 0;
  if ((st = dart_loss_fwd(b, m, c, f, ws, ws_bytes, stream)) != DART_OK) return st;
  total += g_last_launches;
  if ((st = dart_select_steps(f->step_entropy, nullptr, 1, m->S, m, c, f->group_ok, keep, tau, norm, ws, ws_bytes,
                              stream)) != DART_OK)
    return st;
  total += g_last_launches;
  if ((st = dart_loss_bwd(b, m, c, f, keep, norm, dlogits, grad_dtype, ldg, stats, ws, ws_bytes, stream)) != DART_OK)
    return st;
  total += g_last_launches;
  g_last_launches = total;
  return DART_OK;
}

}  // extern "C"
