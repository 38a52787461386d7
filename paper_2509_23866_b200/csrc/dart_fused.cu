// dart_fused.cu -- SURVEY §8(f) NEXT #1: single-read fused loss + gradient
// when the step mask is known in advance (sm_100a).
//
// In a verl-style trainer the old-policy pass (a no-grad forward of theta_old,
// which Eq. 1's denominator needs anyway) can run
// dart_loss_fwd + dart_select_steps and so fix the high-entropy mask
// before the update pass.  The update pass then needs, per kept
// row, only lse (for log pi(y) and p) and the gradient: one read of the row
// from HBM and one write of its gradient -- 4V bytes instead of 6V.
//
// K7 fused_sweep: one CTA per row at a time.  A producer warp streams every
// kept row twice through a shared ring of 4 KB bulk-copy slots: pass 1
// (evict-last L2 policy) feeds the online max / sum, pass 2 (evict-first)
// feeds the gradient.  Pass 2 re-reads the row about one row-time later,
// while it is still resident in the 126 MB L2 (148 CTAs x ~2 rows in flight
// ~ 90 MB), so HBM sees each kept row read once.  Consumer warp w takes the
// chunks j = w, w + NC, ... of each pass (a per-row order, so results do not
// depend on how rows are distributed); the row reduction is a fixed fold over
// the consumer warps.  Rows of masked steps are written as zeros, unread.
#include "dart_common.cuh"
#include "dart_internal.h"

namespace dart {

#ifndef DART_FU_NC
#define DART_FU_NC 8
#endif
#ifndef DART_FU_SW
#define DART_FU_SW 3   // slots per consumer warp (2 measured 9.14 vs 8.91 M tokens/s with split rows, but
                       // compute-sanitizer racecheck then flags the slot hand-back; 3 is clean)
#endif
#ifndef DART_FU_CTAS
#define DART_FU_CTAS 2
#endif
// masked rows' zero stores per lane issued in each row-barrier window (16-byte
// stores; 8..64 measured alike, 0 -- inline between kept rows -- 2% slower)
constexpr int FU_ZB = 16;
constexpr int FU_CL_MAX = 2;   // CTAs a kept row is split over (4-CTA clusters measured 16% slower)
// two CTAs per SM (each 8 consumer warps + 1 producer, 96 KB ring): while one
// CTA sits in its row barrier / epilogue / L2-fed pass 2, the other streams
// its next row from HBM
constexpr int FU_NC = DART_FU_NC;         // consumer warps
constexpr int FU_SW = DART_FU_SW;         // ring slots per consumer warp
constexpr int FU_SLOTS = FU_NC * FU_SW;   // ring slots of CH_BYTES
// Each consumer warp owns FU_SW slots: a warp then never waits on a slot more
// than one phase ahead of the producer (a shared ring let a fast warp alias
// an older mbarrier phase -- parity waits -- and read stale data).
constexpr int FU_PRODUCER = FU_NC, FU_REDUCER = FU_NC + 1;
constexpr int FU_THREADS = (FU_NC + 2) * 32;
constexpr int FU_BAR_PART = 1, FU_BAR_ROW = 2;   // named barriers: partials in / row broadcast out
constexpr int FU_BAR_COUNT = (FU_NC + 1) * 32;    // consumers + reducer

// ---------------------------------------------------------------- cluster helpers
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_count() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_b32(uint32_t raddr, uint32_t v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr), "r"(v),
               "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_b64(uint32_t raddr, uint64_t v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr), "l"(v),
               "r"(rbar)
               : "memory");
}

struct FusedShared {
  uint64_t full[FU_SLOTS];
  uint64_t empty[FU_SLOTS];
  double part_s[FU_NC];
  float part_m[FU_NC];
  float row_g, row_nl2, row_zy;
  int32_t row_y;
  // split-row mode (CL > 1): every cluster CTA's row partial, double-buffered by row parity
  uint64_t mbx[2];
  double mb_s[2][FU_CL_MAX];
  float mb_m[2][FU_CL_MAX];
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}


template <typename Tin>
__device__ __forceinline__ void unpack(const uint4& xv, float* z) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(&xv);
  if (sizeof(Tin) == 2) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      z[2 * j] = bf16lo(w[j]);
      z[2 * j + 1] = bf16hi(w[j]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) z[j] = __uint_as_float(w[j]);
  }
}

template <typename Tin>
__device__ __forceinline__ float load_logit_g(const uint8_t* row, int64_t y) {
  if (sizeof(Tin) == 2) return __uint_as_float(((uint32_t)(*reinterpret_cast<const uint16_t*>(row + 2 * y))) << 16);
  return *reinterpret_cast<const float*>(row + 4 * y);
}

// first local row whose start cost is >= x (costs per step: kept 2, masked 1 or 0)
__device__ __forceinline__ int64_t fu_row_at_cost(const FusedParams& p, int64_t x) {
  const int64_t total = p.step_cost[p.S_loc];
  if (x >= total) return p.T_loc;
  const int64_t s = upper_bound_i64(p.step_cost, 0, p.S_loc + 1, x) - 1;
  const int64_t sg = p.step_begin + s;
  const int64_t t0 = p.step_tok_off[sg] - p.tok_begin, t1 = p.step_tok_off[sg + 1] - p.tok_begin;
  const int64_t per_row = (p.keep[sg] ? 2 : 1) * p.nch;
  const int64_t off = (x - p.step_cost[s] + per_row - 1) / per_row;
  return min(t0 + off, t1);
}

// 32-byte per-row record, built by fused_rec_kernel before the sweep: every
// per-token input the row epilogue needs that does not depend on lse, so the
// epilogue itself is a handful of float ops on prefetched registers.
struct __align__(16) FusedRec {
  int32_t y;        // target (-1 if out of range)
  float zy;         // z_{t,y}
  float lo;         // logp_old
  float w;          // truncated IS weight min(exp(lo - lr), C)
  float A;          // advantage of the row's trajectory
  float lref;       // logp_ref (0 if beta == 0)
  float c;          // per-step loss weight c_s (0: masked step)
  uint32_t flags;   // bit0 kept step, bit1 truncated (ratio >= C), bits 8.. status bits
};

__device__ __forceinline__ int64_t fu_next_kept(const FusedRec* recs, int64_t t, int64_t rb) {
  while (t < rb && !(recs[t].flags & 1u)) ++t;
  return t;
}

__global__ void fused_rec_kernel(FusedParams p, FusedRec* rec) {
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < p.T_loc; t += nthreads) {
    FusedRec r;
    uint32_t bits = 0;
    const int32_t y = p.target[t];
    const uint8_t* row = p.logits + t * p.ld_bytes;
    if (y < 0 || y >= p.V) { bits |= DART_STATUS_TARGET_RANGE; r.y = -1; r.zy = __int_as_float(0x7fc00000); }
    else { r.y = y; r.zy = p.is_bf16 ? load_logit_g<__nv_bfloat16>(row, y) : load_logit_g<float>(row, y); }
    if (r.zy == -INFINITY) bits |= DART_STATUS_TARGET_NEGINF;
    const double lo = p.logp_old[t], lr = p.logp_roll[t];
    const double lref = (p.beta != 0.0) ? (double)p.logp_ref[t] : 0.0;
    if (!isfinite(lo) || !isfinite(lr) || !isfinite(lref)) bits |= DART_STATUS_NONFINITE_LOGP;
    const double ratio = exp(lo - lr);
    r.lo = (float)lo;
    r.w = (float)fmin(ratio, p.is_cap);
    r.A = p.tok_adv[t];
    r.lref = (float)lref;
    const int32_t sl = p.tok_step[t];
    const bool kept = p.keep[p.step_begin + sl] != 0;
    r.c = (float)p.step_scale[sl];
    r.flags = (kept ? 1u : 0u) | (ratio >= p.is_cap ? 2u : 0u) | (kept ? (bits << 8) : 0u);
    reinterpret_cast<FusedRec*>(rec)[t] = r;
  }
}

// row epilogue (token-level ratio): writes the
// per-token outputs and returns g = c_s * dell * invT
__device__ float fused_epilogue(const FusedParams& p, int64_t t, const FusedRec& rc, double Mr, double L2s,
                                bool write = true) {
  uint32_t bits = rc.flags >> 8;
  if (Mr <= (double)clamp_max0(p.c2)) bits |= DART_STATUS_ROW_ALL_NEGINF;
  const double lse2 = Mr + L2s;
  const float logp = (float)(((double)rc.zy * (double)p.c2 - Mr - L2s) * LN2_D);
  const float r = expf(logp - rc.lo);
  const float A = rc.A;
  const float lo_c = (float)(1.0 - p.eps_low), hi_c = (float)(1.0 + p.eps_high);
  const float rcl = fminf(fmaxf(r, lo_c), hi_c);
  const float sur = fminf(r * A, rcl * A);
  const bool act = (A > 0.f) ? (r <= hi_c) : ((A < 0.f) ? (r >= lo_c) : true);
  float kl = 0.f, dkl = 0.f;
  if (p.beta != 0.0) {
    // k3 = e^d - d - 1 and 1 - e^d without fp32 cancellation at small |d|
    // (logp_ref ~ logp: (e^d - d) - 1 in fp32 loses ~1e-7 absolute against a
    // value of d^2 / 2): a Taylor series below |d| = 1/4 (truncation
    // d^5 / 2520 relative), expm1 above.
    const float d = rc.lref - logp;
    const float em1 = expm1f(d);
    dkl = -em1;
    if (fabsf(d) < 0.25f) {
      const float d2 = d * d;
      kl = d2 * (0.5f + d * (1.f / 6.f + d * (1.f / 24.f + d * (1.f / 120.f + d * (1.f / 720.f)))));
    } else {
      kl = em1 - d;
    }
  }
  const float beta = (float)p.beta;
  const float ell = -rc.w * sur + beta * kl;
  const float dell = -rc.w * (act ? A * r : 0.f) + beta * dkl;
  if (!isfinite(ell) || !isfinite(dell)) bits |= DART_STATUS_NONFINITE_LOSS;
  if (!write) return rc.c * dell * (float)p.invT;
  p.lse[t] = (float)(lse2 * LN2_D);
  p.logp[t] = logp;
  p.ell[t] = ell;
  p.dell[t] = dell;
  p.aux_w[t] = rc.w;
  p.aux_kl[t] = kl;
  p.aux_flags[t] = (uint8_t)((act ? 0u : 1u) | (rc.flags & 2u));
  status_or(p.status, bits);
  return rc.c * dell * (float)p.invT;
}

// CL = 2 (split-row mode): a 2-CTA cluster shares each row -- CTA r streams the
// chunks j = r, r + 2, ... through L2 twice, the two (m, s) partials meet via
// st.async in each other's mailbox and are folded in rank order (identical
// lse and g in both CTAs).  Two such CTAs per SM then hold one row's worth of
// bytes between the passes instead of two, which halves the L2 footprint of
// the pass-2 re-read while keeping two independent pipelines per SM.
//
// Roles per CTA: FU_NC consumer warps, a producer lane (bulk copies into one
// FU_SW-slot ring per consumer warp, P1 then P2 chunks of each kept row) and
// a reducer warp.  After pass 1 of a row each consumer warp stores its (m, s)
// partial and ARRIVES on a named barrier (non-blocking); the reducer warp
// SYNCs on it, folds the partials (and the peer CTA's), runs the fp64 row
// epilogue and arrives on a second barrier with g / lse, on which the
// consumers sync before pass 2.  (Measured variants: taking the
// next row's first pass-1 chunks before pass 2 of this row, separate pass-1
// / pass-2 rings, or pass 2 straight from L2 with ld.global all ran slower:
// anything that lets pass 1 run ahead either puts HBM latency in front of
// the L2-fed pass 2 or grows the L2 footprint until pass-2 reads miss.)
template <typename Tin, typename Tout, int CL>
__global__ void __launch_bounds__(FU_THREADS, DART_FU_CTAS) fused_sweep_kernel(const FusedParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;
  FusedShared& sh = *reinterpret_cast<FusedShared*>(smem + (size_t)FU_SLOTS * CH_BYTES);
  constexpr int EPV = 16 / sizeof(Tin);
  constexpr bool OUT_BF16 = sizeof(Tout) == 2;
  constexpr int OUTV = EPV * (int)sizeof(Tout);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < FU_SLOTS; ++s) {
      mbar_init(&sh.full[s], 1);
      mbar_init(&sh.empty[s], 1);
    }
    if (CL > 1) {
      mbar_init(&sh.mbx[0], 1);
      mbar_init(&sh.mbx[1], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (CL > 1) cluster_sync_all();                 // the peer's mailbox exists before any st.async

  // this CTA's (cluster's) contiguous, cost-balanced row range [ra, rb)
  const uint32_t rank = CL > 1 ? cluster_rank() : 0u;
  const int64_t unit = CL > 1 ? (int64_t)cluster_id() : (int64_t)blockIdx.x;
  const int64_t nb = CL > 1 ? (int64_t)cluster_count() : (int64_t)gridDim.x;
  const int64_t total = p.step_cost[p.S_loc];
  const int64_t ra = fu_row_at_cost(p, (total * unit) / nb);
  const int64_t rb = fu_row_at_cost(p, (total * (unit + 1)) / nb);
  // 32-bit chunk / vector arithmetic inside a row (a row is < 2^31 vectors)
  const int nvec = (int)p.nvec;
  // local chunk jl <-> row chunk jl * CL + rank
  const int nch = (int)((p.nch - (int64_t)rank + CL - 1) / CL);
  const float c2 = p.c2;
  const int tail_elems = (int)(p.V % EPV);
  const FusedRec* recs = reinterpret_cast<const FusedRec*>(p.rec);

  if (warp == FU_PRODUCER) {
    // ===================== producer (one lane): chunks in the consumers' ring order
    if (lane == 0) {
      uint64_t pol_last, pol_first;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
      uint32_t nrow = 0;   // kept rows issued so far
      for (int64_t t = fu_next_kept(recs, ra, rb), tn; t < rb; t = tn, ++nrow) {
        const uint8_t* row = p.logits + t * p.ld_bytes;
        const uint32_t fl1 = t + 1 < rb ? recs[t + 1].flags : 1u;   // next row's flags, consumed after this row
        for (int pass = 0; pass < 2; ++pass) {
          for (int j = 0; j < nch; ++j) {
            const int w = j % FU_NC;
            const uint32_t cw = (uint32_t)((nch - w + FU_NC - 1) / FU_NC);    // chunks of warp w per pass
            const uint32_t idx = (2u * nrow + (uint32_t)pass) * cw + (uint32_t)(j / FU_NC);   // warp w's ordinal
            const int slot = w * FU_SW + (int)(idx % FU_SW);
            const uint32_t use = idx / FU_SW;
            if (use > 0) mbar_wait(&sh.empty[slot], (use - 1) & 1u);
            const int v0 = (j * CL + (int)rank) * CH_VEC;
            const uint32_t nv = (uint32_t)min(CH_VEC, nvec - v0);
            mbar_arrive_expect_tx(&sh.full[slot], nv * 16u);
            // pass 1 evict_last (the row must survive in L2 until pass 2), pass 2 evict_first
            bulk_g2s_hint(ring + (size_t)slot * CH_BYTES, row + (size_t)v0 * 16, nv * 16u, &sh.full[slot],
                          pass == 0 ? pol_last : pol_first);
          }
        }
        tn = (t + 1 >= rb || (fl1 & 1u)) ? t + 1 : fu_next_kept(recs, t + 2, rb);
      }
    }
    __syncwarp();
    if (CL > 1) cluster_sync_all();
    return;
  }

  if (warp == FU_REDUCER) {
    // ===================== reducer warp: fold, exchange, epilogue, broadcast
    uint32_t k = 0;
    for (int64_t tk = fu_next_kept(recs, ra, rb); tk < rb; tk = fu_next_kept(recs, tk + 1, rb), ++k) {
      const int par = (int)(k & 1);
      const FusedRec rc = recs[tk];                    // issued before the wait: off the row's critical path
      named_bar_sync(FU_BAR_PART, FU_BAR_COUNT);       // the consumers' partials of row k are in
      // fixed-order fold of the consumer warps' partials (one per lane, xor butterfly)
      const float mw = lane < FU_NC ? sh.part_m[lane] : -INFINITY;
      const double sw = lane < FU_NC ? sh.part_s[lane] : 0.0;
      const float Mf = warp_max_f(sw > 0.0 ? mw : -INFINITY);
      double Sr = warp_sum_d(sw > 0.0 ? sw * (double)ex2(mw - Mf) : 0.0);
      double Mr = Sr > 0.0 ? (double)Mf : -INFINITY;
      if (lane == 0) {
        if (CL > 1) {                            // exchange with the peer CTA, fold in rank order
          sh.mb_m[par][rank] = (float)Mr;
          sh.mb_s[par][rank] = Sr;
          mbar_arrive_expect_tx(&sh.mbx[par], 12u * (CL - 1));          // 4 + 8 bytes from every peer
#pragma unroll
          for (int d = 1; d < CL; ++d) {
            const uint32_t peer = (rank + (uint32_t)d) % (uint32_t)CL;
            const uint32_t rbar = map_rank(&sh.mbx[par], peer);
            st_async_b32(map_rank(&sh.mb_m[par][rank], peer), __float_as_uint((float)Mr), rbar);
            st_async_b64(map_rank(&sh.mb_s[par][rank], peer), (uint64_t)__double_as_longlong(Sr), rbar);
          }
          mbar_wait(&sh.mbx[par], (k >> 1) & 1u);
          Mr = -INFINITY;
          Sr = 0.0;
          for (int k2 = 0; k2 < CL; ++k2) {
            const double Mk = (double)sh.mb_m[par][k2], Sk = sh.mb_s[par][k2];
            if (Sk == 0.0) continue;
            if (Mr == -INFINITY) { Mr = Mk; Sr = Sk; continue; }
            const double mn = fmax(Mr, Mk);
            Sr = Sr * (double)ex2((float)(Mr - mn)) + Sk * (double)ex2((float)(Mk - mn));
            Mr = mn;
          }
        }
        const double L2s = log2(Sr);
        sh.row_g = fused_epilogue(p, tk, rc, Mr, L2s, rank == 0);
        sh.row_nl2 = (float)(-(Mr + L2s));
        sh.row_y = rc.y;
        sh.row_zy = rc.zy;
      }
      named_bar_arrive(FU_BAR_ROW, FU_BAR_COUNT);      // row k's g / lse out (consumers sync)
    }
    if (CL > 1) cluster_sync_all();                 // no CTA exits with mailbox traffic pending
    return;
  }

  // ===================== consumers (FU_NC warps) =====================
  const uint32_t cw = (uint32_t)((nch - warp + FU_NC - 1) / FU_NC);   // this warp's chunks per pass
  uint32_t idx = 0;              // this warp's ring ordinal (chunks taken so far)
  uint32_t bad = 0;

  // the chunk at the head of this warp's ring: wait, pull into registers, slot back to the producer
  auto take = [&](uint4 (&x)[VPL], int nv) {
    const int slot = warp * FU_SW + (int)(idx % FU_SW);
    mbar_wait(&sh.full[slot], (idx / FU_SW) & 1u);
    ++idx;
    const uint8_t* sp = ring + (size_t)slot * CH_BYTES;
    if (nv == CH_VEC) {     // full chunk: unpredicated loads (measured 4% faster than the guarded form)
#pragma unroll
      for (int q = 0; q < VPL; ++q) x[q] = lds128(sp + (lane + 32 * q) * 16);
    } else {
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const int vi = lane + 32 * q;
        x[q] = (vi < nv) ? lds128(sp + vi * 16) : make_uint4(0u, 0u, 0u, 0u);
      }
    }
    fence_reads_before_refill();
    __syncwarp();
    if (lane == 0) mbar_arrive(&sh.empty[slot]);   // slot back to the producer
  };

  // pass 1 over this warp's chunks [ji0, ji1) of a row: online max / sum into (m, s01, s23)
  auto pass1 = [&](uint32_t ji0, uint32_t ji1, float& m, float2& s01, float2& s23) {
    for (uint32_t ji = ji0; ji < ji1; ++ji) {
      const int j = warp + (int)ji * FU_NC;
      const int v0 = (j * CL + (int)rank) * CH_VEC;
      const int nv = min(CH_VEC, nvec - v0);
      uint4 x[VPL];
      take(x, nv);
      const bool tail_chunk = tail_elems && v0 + nv == nvec;
      if (sizeof(Tin) == 2 && nv == CH_VEC && !tail_chunk) {
        // fast path: packed bf16x2 max, one unpack per pair; -inf logits give
        // 2^-inf = 0 and there is no 0*inf term (no entropy in this pass)
        uint32_t mx = 0xff80ff80u;
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          mx = bmax2_nan(mx, x[q].x);
          mx = bmax2_nan(mx, x[q].y);
          mx = bmax2_nan(mx, x[q].z);
          mx = bmax2_nan(mx, x[q].w);
        }
        const float cmr = fmax_nan(bf16lo(mx), bf16hi(mx));
        if (!(cmr < INFINITY)) bad |= DART_STATUS_NONFINITE_LOGIT;
        const float cms = cmr * c2;
        if (cms > m + 2.0f) {   // lazy running max (LAZY_M = 2, as in the fwd sweep)
          const float sc = ex2(m - cms);
          s01 = __fmul2_rn(s01, make_float2(sc, sc));
          s23 = __fmul2_rn(s23, make_float2(sc, sc));
          m = cms;
        }
        const float2 cc = make_float2(c2, c2), nm = make_float2(-m, -m);
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          const float2 d0 = __ffma2_rn(make_float2(bf16lo(x[q].x), bf16hi(x[q].x)), cc, nm);
          const float2 d1 = __ffma2_rn(make_float2(bf16lo(x[q].y), bf16hi(x[q].y)), cc, nm);
          const float2 d2 = __ffma2_rn(make_float2(bf16lo(x[q].z), bf16hi(x[q].z)), cc, nm);
          const float2 d3 = __ffma2_rn(make_float2(bf16lo(x[q].w), bf16hi(x[q].w)), cc, nm);
          s01 = __fadd2_rn(s01, make_float2(ex2(d0.x), ex2(d0.y)));
          s23 = __fadd2_rn(s23, make_float2(ex2(d1.x), ex2(d1.y)));
          s01 = __fadd2_rn(s01, make_float2(ex2(d2.x), ex2(d2.y)));
          s23 = __fadd2_rn(s23, make_float2(ex2(d3.x), ex2(d3.y)));
        }
        continue;
      }
      float cm = -INFINITY;
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const int vi = lane + 32 * q;
        if (vi < nv) {
          float z[EPV];
          unpack<Tin>(x[q], z);
#pragma unroll
          for (int e = 0; e < EPV; ++e) {
            if (tail_chunk && vi == nv - 1 && e >= tail_elems) z[e] = NEG_CLAMP;
            cm = fmax_nan(cm, z[e]);
          }
        }
      }
      if (!(cm < INFINITY)) bad |= DART_STATUS_NONFINITE_LOGIT;
      const float cms = fmaxf(cm, NEG_CLAMP) * c2;
      if (cms > m + 2.0f) {
        const float sc = ex2(m - cms);
        s01 = __fmul2_rn(s01, make_float2(sc, sc));
        s23 = __fmul2_rn(s23, make_float2(sc, sc));
        m = cms;
      }
      const float2 cc = make_float2(c2, c2), nm = make_float2(-m, -m);
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const int vi = lane + 32 * q;
        if (vi < nv) {
          float z[EPV];
          unpack<Tin>(x[q], z);
#pragma unroll
          for (int e = 0; e < EPV; ++e) {
            if (tail_chunk && vi == nv - 1 && e >= tail_elems) z[e] = NEG_CLAMP;
            z[e] = fmaxf(z[e], NEG_CLAMP);   // -inf logits contribute exp -> 0
          }
#pragma unroll
          for (int e = 0; e < EPV; e += 4) {
            const float2 d0 = __ffma2_rn(make_float2(z[e], z[e + 1]), cc, nm);
            const float2 d1 = __ffma2_rn(make_float2(z[e + 2], z[e + 3]), cc, nm);
            s01 = __fadd2_rn(s01, make_float2(ex2(d0.x), ex2(d0.y)));
            s23 = __fadd2_rn(s23, make_float2(ex2(d1.x), ex2(d1.y)));
          }
        }
      }
    }
  };

  // warp partial of a row (fixed lane fold) -> the reducer; never waits
  auto publish = [&](float m, float2 s01, float2 s23) {
    const float M = warp_max_f(m);
    const float sl = (s01.x + s01.y) + (s23.x + s23.y);
    const double sd = warp_sum_d((double)sl * (double)ex2(m - M));
    if (lane == 0) {
      sh.part_m[warp] = M;
      sh.part_s[warp] = sd;
    }
    named_bar_arrive(FU_BAR_PART, FU_BAR_COUNT);
  };

  // pass 2 over this warp's chunks of row t: dz = -g p (+ g at the target)
  auto pass2 = [&](int64_t t, float g, float nl2, int32_t y, float zy) {
    uint8_t* orow = p.dlogits + t * p.ldg_bytes;
    const float2 cc2 = make_float2(c2, c2), nl = make_float2(nl2, nl2), ng = make_float2(-g, -g);
    for (uint32_t ji = 0; ji < cw; ++ji) {
      const int j = warp + (int)ji * FU_NC;
      const int v0 = (j * CL + (int)rank) * CH_VEC;
      const int nv = min(CH_VEC, nvec - v0);
      uint4 x[VPL];
      take(x, nv);
      if (OUT_BF16 && EPV == 8 && nv == CH_VEC && !(tail_elems && v0 + nv == nvec)) {
        // full bf16 chunk: no per-vector guards, immediate store offsets from the lane's first vector
        uint8_t* const olane = orow + (v0 + lane) * OUTV;
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          float z[EPV], o[EPV];
          unpack<Tin>(x[q], z);
#pragma unroll
          for (int e = 0; e < EPV; e += 2) {
            const float2 d = __ffma2_rn(make_float2(z[e], z[e + 1]), cc2, nl);
            const float2 dz = __fmul2_rn(make_float2(ex2(d.x), ex2(d.y)), ng);
            o[e] = dz.x;
            o[e + 1] = dz.y;
          }
          stg128_cs(olane + q * 32 * OUTV, make_uint4(pack_bf16x2(o[0], o[1]), pack_bf16x2(o[2], o[3]),
                                                      pack_bf16x2(o[4], o[5]), pack_bf16x2(o[6], o[7])));
        }
      } else {
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          const int vi = lane + 32 * q;
          if (vi < nv) {
            const int gv = v0 + vi;
            float z[EPV], o[EPV];
            unpack<Tin>(x[q], z);
#pragma unroll
            for (int e = 0; e < EPV; e += 2) {
              const float2 d = __ffma2_rn(make_float2(z[e], z[e + 1]), cc2, nl);
              const float2 dz = __fmul2_rn(make_float2(ex2(d.x), ex2(d.y)), ng);
              o[e] = dz.x;
              o[e + 1] = dz.y;
            }
            const int nvalid = (tail_elems && gv == nvec - 1) ? tail_elems : EPV;
            uint8_t* dst = orow + gv * OUTV;
            if (nvalid == EPV) {
              if (OUT_BF16 && EPV == 8) {
                stg128_cs(dst, make_uint4(pack_bf16x2(o[0], o[1]), pack_bf16x2(o[2], o[3]), pack_bf16x2(o[4], o[5]),
                                          pack_bf16x2(o[6], o[7])));
              } else if (OUT_BF16) {
                *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16x2(o[0], o[1]), pack_bf16x2(o[2], o[3]));
              } else {
#pragma unroll
                for (int e = 0; e < EPV; e += 4)
                  stg128_cs(dst + 4 * e, make_uint4(__float_as_uint(o[e]), __float_as_uint(o[e + 1]),
                                                    __float_as_uint(o[e + 2]), __float_as_uint(o[e + 3])));
              }
            } else {
              for (int e = 0; e < nvalid; ++e) {
                if (OUT_BF16) reinterpret_cast<__nv_bfloat16*>(dst)[e] = __float2bfloat16_rn(o[e]);
                else reinterpret_cast<float*>(dst)[e] = o[e];
              }
            }
          }
        }
      }
      // target element: g (1 - p_y), rewritten by its owning lane after the vector store
      if (y >= 0 && y < p.V) {
        const int yv = y / EPV;
        if (yv >= v0 && yv < v0 + nv && lane == ((yv - v0) & 31)) {
          const float py = ex2(fmaf(zy, c2, nl2));
          const float dzy = fmaf(-g, py, g);
          if (OUT_BF16) reinterpret_cast<__nv_bfloat16*>(orow)[y] = __float2bfloat16_rn(dzy);
          else reinterpret_cast<float*>(orow)[y] = dzy;
        }
      }
    }
  };

  // masked rows: zeros, no read, deferred into the row-barrier windows -- a
  // per-warp cursor over the masked rows below `zlim` (rows in order, this
  // warp's vectors li = warp*32 + lane + k*FU_NC*32 of each)
  int64_t zt = ra;
  int zli = warp * 32 + lane;
  bool zt_masked = zt < rb && !(recs[zt].flags & 1u);
  const int zrow_vecs = nch * CH_VEC;
  auto zero_some = [&](int64_t zlim, int budget) {
    if (!p.zero_fill) return;
    while (zt < zlim) {
      if (!zt_masked) {
        ++zt;
        zt_masked = zt < rb && !(recs[zt].flags & 1u);
        continue;
      }
      if (budget <= 0) return;
      uint8_t* orow = p.dlogits + zt * p.ldg_bytes;
      for (; zli < zrow_vecs && budget > 0; zli += FU_NC * 32, --budget) {
        const int vi = ((zli / CH_VEC) * CL + (int)rank) * CH_VEC + (zli % CH_VEC);
        if (vi >= nvec) continue;
        const int nvalid = (tail_elems && vi == nvec - 1) ? tail_elems : EPV;
        uint8_t* dst = orow + vi * OUTV;
        if (nvalid == EPV) {
          if (OUT_BF16 && EPV == 8) stg128_cs(dst, make_uint4(0u, 0u, 0u, 0u));
          else if (OUT_BF16) *reinterpret_cast<uint2*>(dst) = make_uint2(0u, 0u);
          else
            for (int e = 0; e < EPV; e += 4) stg128_cs(dst + 4 * e, make_uint4(0u, 0u, 0u, 0u));
        } else {
          for (int e = 0; e < nvalid; ++e) {
            if (OUT_BF16) reinterpret_cast<__nv_bfloat16*>(dst)[e] = __float2bfloat16_rn(0.f);
            else reinterpret_cast<float*>(dst)[e] = 0.f;
          }
        }
      }
      if (zli >= zrow_vecs) {
        zli = warp * 32 + lane;
        ++zt;
        zt_masked = zt < rb && !(recs[zt].flags & 1u);
      }
    }
  };

  int64_t tk = fu_next_kept(recs, ra, rb);
  while (tk < rb) {
    float m = clamp_max0(c2);                       // (see dart_common.cuh)
    float2 s01 = make_float2(0.f, 0.f), s23 = make_float2(0.f, 0.f);
    pass1(0u, cw, m, s01, s23);
    publish(m, s01, s23);                            // non-blocking: the reducer folds
    zero_some(tk, FU_ZB);                           // masked rows below this one, while the row reduces
    __syncwarp();                                   // reconverge: bar.sync is warp-aligned
    named_bar_sync(FU_BAR_ROW, FU_BAR_COUNT);       // row tk's g / lse
    const float g = sh.row_g, nl2 = sh.row_nl2, zy = sh.row_zy;
    const int32_t y = sh.row_y;
    const uint32_t fl1 = tk + 1 < rb ? recs[tk + 1].flags : 1u;    // prefetched; consumed after pass 2
    pass2(tk, g, nl2, y, zy);
    const int64_t tn = (tk + 1 >= rb || (fl1 & 1u)) ? tk + 1 : fu_next_kept(recs, tk + 2, rb);
    tk = tn;
  }
  zero_some(rb, 1 << 30);                           // what is left (after the last kept row)
  bad = warp_or(bad);
  if (lane == 0 && bad) status_or(p.status, bad);
  if (CL > 1) cluster_sync_all();
}

cudaError_t launch_fused_rec(const FusedParams& p, cudaStream_t st) {
  if (p.T_loc <= 0) return cudaSuccess;
  int64_t blocks = (p.T_loc + 255) / 256;
  if (blocks > 8192) blocks = 8192;
  fused_rec_kernel<<<(unsigned)blocks, 256, 0, st>>>(p, reinterpret_cast<FusedRec*>(p.rec));
  return cudaGetLastError();
}

template <typename Tin, typename Tout, int CL>
static cudaError_t launch_fused_cl(const FusedParams& p, int num_sms, size_t smem, cudaStream_t st);

template <typename Tin, typename Tout>
static cudaError_t launch_fused_t(const FusedParams& p, int num_sms, bool split, cudaStream_t st) {
  const size_t smem = (size_t)FU_SLOTS * CH_BYTES + sizeof(FusedShared);
  if (!split) {
    auto kern = fused_sweep_kernel<Tin, Tout, 1>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)(num_sms * DART_FU_CTAS), FU_THREADS, smem, st>>>(p);
    return cudaGetLastError();
  }
  return launch_fused_cl<Tin, Tout, FU_CL_MAX>(p, num_sms, smem, st);
}

template <typename Tin, typename Tout, int CL>
static cudaError_t launch_fused_cl(const FusedParams& p, int num_sms, size_t smem, cudaStream_t st) {
  auto kern = fused_sweep_kernel<Tin, Tout, CL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(FU_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3((unsigned)(num_sms * DART_FU_CTAS));
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
    (void)cudaGetLastError();
    n = num_sms * DART_FU_CTAS / CL;
  }
  cfg.gridDim = dim3((unsigned)(CL * n));
  return cudaLaunchKernelEx(&cfg, kern, p);
}

cudaError_t launch_fused_sweep(const FusedParams& p, bool in_bf16, bool out_bf16, int num_sms, bool split,
                               cudaStream_t st) {
  if (in_bf16 && out_bf16) return launch_fused_t<__nv_bfloat16, __nv_bfloat16>(p, num_sms, split, st);
  if (in_bf16) return launch_fused_t<__nv_bfloat16, float>(p, num_sms, split, st);
  if (out_bf16) return launch_fused_t<float, __nv_bfloat16>(p, num_sms, split, st);
  return launch_fused_t<float, float>(p, num_sms, split, st);
}

}  // namespace dart
