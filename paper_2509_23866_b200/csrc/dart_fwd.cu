// dart_fwd.cu -- forward half of the DART loss pass (sm_100a).
//
//   K0a adv_kernel      per group g: step-weighted mean / population std of R
//                       over the step group D_g,
//                       A_i, group_ok; plus metadata validation.
//   K0b tok_meta_kernel per local step: token -> (local step, A) tables.
//   K1  fwd_sweep       THE HOT LOOP: one streamed read of every logit row
//                       (bulk copies into a per-warp shared-memory ring),
//                       online max / sum / entropy in the log2 domain, then
//                       the fused epilogue: lse, log pi(y),
//                       H, IS weight, clipped
//                       surrogate and k3 KL (Eq. 1/2).
//   K2  step_reduce     per local step: mean entropy and the
//                       fixed-order sums the loss / statistics need.
#include "dart_common.cuh"
#include "dart_internal.h"

namespace dart {

// ============================================================== K0a
__global__ void adv_kernel(AdvParams p) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  uint32_t bits = 0;
  // --- per group (one thread per group; groups have <= a few dozen trajectories)
  for (int64_t g = tid; g < p.G; g += nthreads) {
    const int64_t i0 = lower_bound_i32(p.traj_group, 0, p.N_traj, g);
    const int64_t i1 = lower_bound_i32(p.traj_group, i0, p.N_traj, g + 1);
    p.grp_traj[g] = i0;
    if (g == p.G - 1) p.grp_traj[p.G] = i1;
    double sumL = 0.0, sumLR = 0.0;
    bool all_equal = true;
    float R0 = 0.f;
    bool have = false;
    for (int64_t i = i0; i < i1; ++i) {
      const double L = (double)(p.traj_step_off[i + 1] - p.traj_step_off[i]);
      if (L <= 0) continue;
      const float R = p.traj_reward[i];
      if (!have) { R0 = R; have = true; } else if (R != R0) all_equal = false;
      sumL += L;
      sumLR += L * (double)R;
    }
    uint8_t ok = 0;
    if (sumL > 0) {
      // PAPER.md:134; all rewards equal: R itself (exact arithmetic -- the
      // rounded quotient's residue would become A = residue / adv_eps)
      const double Rbar = all_equal ? (double)R0 : sumLR / sumL;
      double var = 0.0;
      for (int64_t i = i0; i < i1; ++i) {
        const double L = (double)(p.traj_step_off[i + 1] - p.traj_step_off[i]);
        if (L <= 0) continue;
        const double d = (double)p.traj_reward[i] - Rbar;
        var += L * d * d;
      }
      var /= sumL;                                            // PAPER.md:135 (population)
      double sigma = all_equal ? 0.0 : sqrt(var);
      if (p.adv_eps > 0.0) {
        ok = 1;
        for (int64_t i = i0; i < i1; ++i) p.adv[i] = (float)(((double)p.traj_reward[i] - Rbar) / (sigma + p.adv_eps));
      } else if (sigma > 0.0) {
        ok = 1;
        for (int64_t i = i0; i < i1; ++i) p.adv[i] = (float)(((double)p.traj_reward[i] - Rbar) / sigma);
      } else {
        for (int64_t i = i0; i < i1; ++i) p.adv[i] = 0.f;    // group skipped
      }
    } else {
      for (int64_t i = i0; i < i1; ++i) p.adv[i] = 0.f;
    }
    p.group_ok[g] = ok;
  }
  // --- metadata validation (global CSR)
  for (int64_t i = tid; i < p.N_traj; i += nthreads) {
    const int64_t a = p.traj_step_off[i], b = p.traj_step_off[i + 1];
    if (b < a) bits |= DART_STATUS_BAD_CSR;
    if (b == a) bits |= DART_STATUS_EMPTY;
    const int32_t gi = p.traj_group[i];
    if (gi < 0 || gi >= p.G) bits |= DART_STATUS_BAD_CSR;
    if (i + 1 < p.N_traj && p.traj_group[i + 1] < gi) bits |= DART_STATUS_BAD_CSR;
  }
  for (int64_t s = tid; s < p.S; s += nthreads) {
    const int64_t a = p.step_tok_off[s], b = p.step_tok_off[s + 1];
    if (b < a) bits |= DART_STATUS_BAD_CSR;
    if (b == a) bits |= DART_STATUS_EMPTY;
  }
  if (tid == 0) {
    if (p.traj_step_off[0] != 0 || p.traj_step_off[p.N_traj] != p.S || p.step_tok_off[0] != 0 ||
        p.step_tok_off[p.S] != p.T)
      bits |= DART_STATUS_BAD_CSR;
  }
  status_or(p.status, bits);
}

// ============================================================== K0b
// One warp per local step: fills tok_adv[t] = A_{traj(s)} and tok_step[t] = s_loc.
__global__ void tok_meta_kernel(TokMetaParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t bits = 0;
  if (w == 0 && lane == 0) {
    if (p.step_begin < 0 || p.step_begin + p.S_loc > p.S ||
        p.step_tok_off[p.step_begin] != p.tok_begin ||
        p.step_tok_off[p.step_begin + p.S_loc] != p.tok_begin + p.T_loc)
      bits |= DART_STATUS_BAD_CSR;
  }
  for (int64_t s = w; s < p.S_loc; s += nw) {
    const int64_t sg = p.step_begin + s;
    const int64_t t0 = p.step_tok_off[sg] - p.tok_begin;
    const int64_t t1 = p.step_tok_off[sg + 1] - p.tok_begin;
    if (t0 < 0 || t1 > p.T_loc || t1 < t0) { bits |= DART_STATUS_BAD_CSR; continue; }
    const int64_t i = upper_bound_i64(p.traj_step_off, 0, p.N_traj + 1, sg) - 1;
    const float A = (i >= 0 && i < p.N_traj) ? p.adv[i] : 0.f;
    for (int64_t t = t0 + lane; t < t1; t += 32) {
      p.tok_adv[t] = A;
      p.tok_step[t] = (int32_t)s;
    }
  }
  status_or(p.status, bits);
}

// ============================================================== K1 helpers
// Canonical row decomposition: KSEG segments whose boundaries are multiples of
// the chunk (FCH_VEC vectors) -- only the row's last chunk can be partial.  The
// per-row reduction order (lane <- vector mod 32, chunk-wise max update,
// segment partials folded left to right) depends only on nvec, never on how
// rows or segments are distributed over warps.
constexpr int FVPL = FCH_VEC / 32;   // 16-byte vectors per lane per fwd chunk
__device__ __forceinline__ int64_t seg_begin(int64_t nvec, int k) {
  if (k >= KSEG) return nvec;
  return ((nvec * k) / KSEG) & ~(int64_t)(FCH_VEC - 1);
}

// Work stream of one warp: units u = wid, wid+W, ...; unit = (row, part);
// part p covers segments [p*KSEG/nsplit, (p+1)*KSEG/nsplit) (nsplit = 2^lg).
// Row-relative vector indices are 32-bit (rows < 2^31 vectors); the common
// step (next chunk in the same segment) is a few integer ops, transitions are
// out of line.
struct Stream {
  int64_t u, row;
  int32_t v, vend, k, kend;
  bool valid;
};

__device__ __forceinline__ void stream_set_unit(Stream& s, int64_t uu, int64_t units, int lg, int64_t nvec) {
  s.u = uu;
  s.valid = uu < units;
  if (!s.valid) return;
  s.row = uu >> lg;
  const int part = (int)(uu & ((1 << lg) - 1));
  int k = (part * KSEG) >> lg;
  s.kend = ((part + 1) * KSEG) >> lg;
  s.v = (int32_t)seg_begin(nvec, k);
  int32_t ve = (int32_t)seg_begin(nvec, k + 1);
  while (s.v == ve && k + 1 < s.kend) { ++k; ve = (int32_t)seg_begin(nvec, k + 1); }  // skip empty segments
  s.k = k;
  s.vend = ve;
}

// called when the chunk just taken ended segment s.k: move to the next
// non-empty segment of the unit or to the next unit; returns unit_end
__device__ __forceinline__ bool stream_next_segment(Stream& s, int64_t W, int64_t units, int lg, int64_t nvec) {
  int kk = s.k + 1;
  int32_t ve = s.vend;
  while (kk < s.kend) {
    ve = (int32_t)seg_begin(nvec, kk + 1);
    if (ve > s.v) break;
    ++kk;
  }
  if (kk >= s.kend) {
    stream_set_unit(s, s.u + W, units, lg, nvec);
    return true;
  }
  s.k = kk;
  s.vend = ve;
  return false;
}

// Lazy running max (log2 units): a lane rescales only when a chunk's max
// exceeds its reference by more than LAZY_M.  The shift then sits up to LAZY_M
// below the true max, so u = sum e (x-m) mixes signs; the extra fp32 error in
// H is ~LAZY_M * eps relative -- 2 keeps it far below the 1e-5 bar (64 did not).
constexpr float LAZY_M = 2.0f;

// per-lane online state (log2 domain)
struct LaneAcc {
  float m;
  float2 s[4], u[4];
};

__device__ __forceinline__ void acc_reset(LaneAcc& a, float m0) {
  a.m = m0;
#pragma unroll
  for (int j = 0; j < 4; ++j) { a.s[j] = make_float2(0.f, 0.f); a.u[j] = make_float2(0.f, 0.f); }
}

__device__ __forceinline__ void acc_rescale(LaneAcc& a, float mnew) {
  const float dm = a.m - mnew;           // <= 0, finite
  const float sc = ex2(dm);
  const float2 dm2 = make_float2(dm, dm), sc2 = make_float2(sc, sc);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    a.u[j] = __fmul2_rn(__ffma2_rn(a.s[j], dm2, a.u[j]), sc2);
    a.s[j] = __fmul2_rn(a.s[j], sc2);
  }
  a.m = mnew;
}

// accumulate one pair of logits (already in f32) into accumulator j
__device__ __forceinline__ void acc_pair(LaneAcc& a, int j, float2 z, float2 cc, float2 nm) {
  const float2 d = __ffma2_rn(z, cc, nm);
  const float2 e = make_float2(ex2(d.x), ex2(d.y));
  a.s[j] = __fadd2_rn(a.s[j], e);
  a.u[j] = __ffma2_rn(e, d, a.u[j]);
}

// ------------------------------------------------------------ chunk bodies
// bf16: one 16-byte vector = 8 logits = 4 bf16x2 words
template <bool FULL>
__device__ __forceinline__ void chunk_bf16(uint4 (&x)[FVPL], int nv, int lane, float c2, LaneAcc& a,
                                           uint32_t& bad, int tail_idx, uint32_t tail_keep_mask) {
  if (!FULL) {
#pragma unroll
    for (int k = 0; k < FVPL; ++k)
      if (lane + 32 * k >= nv) x[k] = make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u);
  }
  if (tail_idx >= 0) {  // last vector of the row: logits >= V are not part of the row
#pragma unroll
    for (int k = 0; k < FVPL; ++k) {
      if (lane + 32 * k == tail_idx) {
        uint32_t* w = reinterpret_cast<uint32_t*>(&x[k]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t lo_ok = (tail_keep_mask >> (2 * j)) & 1u, hi_ok = (tail_keep_mask >> (2 * j + 1)) & 1u;
          w[j] = (lo_ok ? (w[j] & 0x0000ffffu) : NEG_CLAMP_BF16) | (hi_ok ? (w[j] & 0xffff0000u) : (NEG_CLAMP_BF16 << 16));
        }
      }
    }
  }
  uint32_t mx = 0xff80ff80u;
#pragma unroll
  for (int k = 0; k < FVPL; ++k) {
    mx = bmax2_nan(mx, x[k].x);
    mx = bmax2_nan(mx, x[k].y);
    mx = bmax2_nan(mx, x[k].z);
    mx = bmax2_nan(mx, x[k].w);
  }
  const float cmr = fmax_nan(bf16lo(mx), bf16hi(mx));
  if (!(cmr < INFINITY)) bad |= DART_STATUS_NONFINITE_LOGIT;      // NaN or +inf
  // lazy running max (see LAZY_M)
  const float cm = cmr * c2;
  if (__any_sync(0xffffffffu, cm > a.m + LAZY_M)) acc_rescale(a, (cm > a.m + LAZY_M) ? cm : a.m);
  const float2 cc = make_float2(c2, c2), nm = make_float2(-a.m, -a.m);
#pragma unroll
  for (int k = 0; k < FVPL; ++k) {
    if (FULL || lane + 32 * k < nv) {
      acc_pair(a, 0, make_float2(bf16lo(x[k].x), bf16hi(x[k].x)), cc, nm);
      acc_pair(a, 1, make_float2(bf16lo(x[k].y), bf16hi(x[k].y)), cc, nm);
      acc_pair(a, 2, make_float2(bf16lo(x[k].z), bf16hi(x[k].z)), cc, nm);
      acc_pair(a, 3, make_float2(bf16lo(x[k].w), bf16hi(x[k].w)), cc, nm);
    }
  }
}

// f32: one vector = 4 logits
template <bool FULL>
__device__ __forceinline__ void chunk_f32(const uint4 (&xr)[FVPL], int nv, int lane, float c2, LaneAcc& a,
                                          uint32_t& bad, int tail_idx, uint32_t tail_keep_mask) {
  float4 x[FVPL];
#pragma unroll
  for (int k = 0; k < FVPL; ++k) {
    const int vi = lane + 32 * k;
    if (FULL || vi < nv) {
      x[k] = make_float4(__uint_as_float(xr[k].x), __uint_as_float(xr[k].y), __uint_as_float(xr[k].z),
                         __uint_as_float(xr[k].w));
    } else {
      x[k] = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    }
  }
  if (tail_idx >= 0) {
#pragma unroll
    for (int k = 0; k < FVPL; ++k) {
      if (lane + 32 * k == tail_idx) {
        if (!((tail_keep_mask >> 0) & 1u)) x[k].x = NEG_CLAMP;
        if (!((tail_keep_mask >> 1) & 1u)) x[k].y = NEG_CLAMP;
        if (!((tail_keep_mask >> 2) & 1u)) x[k].z = NEG_CLAMP;
        if (!((tail_keep_mask >> 3) & 1u)) x[k].w = NEG_CLAMP;
      }
    }
  }
  float cmr = -INFINITY;
#pragma unroll
  for (int k = 0; k < FVPL; ++k) {
    cmr = fmax_nan(cmr, x[k].x);
    cmr = fmax_nan(cmr, x[k].y);
    cmr = fmax_nan(cmr, x[k].z);
    cmr = fmax_nan(cmr, x[k].w);
  }
  if (!(cmr < INFINITY)) bad |= DART_STATUS_NONFINITE_LOGIT;
  // lazy running max (see LAZY_M)
  const float cm = cmr * c2;
  if (__any_sync(0xffffffffu, cm > a.m + LAZY_M)) acc_rescale(a, (cm > a.m + LAZY_M) ? cm : a.m);
  const float2 cc = make_float2(c2, c2), nm = make_float2(-a.m, -a.m);
#pragma unroll
  for (int k = 0; k < FVPL; ++k) {
    if (FULL || lane + 32 * k < nv) {
      acc_pair(a, 0, make_float2(x[k].x, x[k].y), cc, nm);
      acc_pair(a, 1, make_float2(x[k].z, x[k].w), cc, nm);
    }
  }
}

// Slow path for a segment that contained -inf logits (0 * -inf made u NaN):
// re-read the segment from global with -inf clamped to NEG_CLAMP, two passes.
template <typename Tin>
__device__ Part segment_slow(const FwdParams& p, int64_t row, int k, int lane) {
  const int64_t vb = seg_begin(p.nvec, k), ve = seg_begin(p.nvec, k + 1);
  constexpr int EPV = 16 / sizeof(Tin);
  const Tin* base = reinterpret_cast<const Tin*>(p.logits + row * p.ld_bytes);
  const int64_t e0 = vb * EPV, e1 = min(ve * EPV, p.V);
  float m = NEG_CLAMP * p.c2;
  for (int64_t e = e0 + lane; e < e1; e += 32) {
    float z = fmaxf((float)base[e], NEG_CLAMP);
    m = fmaxf(m, z * p.c2);
  }
  const float M = warp_max_f(m);
  double s = 0.0, u = 0.0;
  for (int64_t e = e0 + lane; e < e1; e += 32) {
    float z = fmaxf((float)base[e], NEG_CLAMP);
    const float d = fmaf(z, p.c2, -M);
    const float ee = ex2(d);
    s += (double)ee;
    u += (double)ee * (double)d;
  }
  Part r;
  r.m = (double)M;
  r.s = warp_sum_d(s);
  r.u = warp_sum_d(u);
  return r;
}

__device__ __forceinline__ float load_logit(const FwdParams& p, int64_t row, int64_t y, bool is_bf16) {
  const uint8_t* rp = p.logits + row * p.ld_bytes;
  if (is_bf16) {
    const uint16_t b = *reinterpret_cast<const uint16_t*>(rp + 2 * y);
    return __uint_as_float(((uint32_t)b) << 16);
  }
  return *reinterpret_cast<const float*>(rp + 4 * y);
}

// Row epilogue: everything per token that needs the full row (all lanes
// compute redundantly; lane 0 writes).  Double precision: once per 152K logits.
// zy: the target's logit (NaN with DART_STATUS_TARGET_RANGE already in bits
// when y is out of range).  Shared by the logits sweep and the LM-head path.
__device__ void row_epilogue_z(const FwdParams& p, int64_t row, Part R, uint32_t bits, float zy, int lane) {
  const double lo = p.logp_old[row], lr = p.logp_roll[row];
  const double lref = (p.beta != 0.0) ? (double)p.logp_ref[row] : 0.0;
  const double A = p.tok_adv[row];
  if (!isfinite(lo) || !isfinite(lr) || !isfinite(lref)) bits |= DART_STATUS_NONFINITE_LOGP;
  if (zy == -INFINITY) bits |= DART_STATUS_TARGET_NEGINF;
  if (R.m <= (double)(NEG_CLAMP * p.c2)) bits |= DART_STATUS_ROW_ALL_NEGINF;

  const double L2s = log2(R.s);
  const double lse2 = R.m + L2s;                               // log2 sum 2^(z c2)
  const double lse = lse2 * LN2_D;
  double H = LN2_D * (L2s - R.u / R.s);                        // PAPER.md:238, nats
  if (H < 0.0) H = 0.0;
  const double logp = ((double)zy * (double)p.c2 - R.m - L2s) * LN2_D;   // log pi(y)
  // token-level ratio and truncated IS weight
  const double r = exp(logp - lo);
  const double ratio = exp(lo - lr);
  const double w = fmin(ratio, p.is_cap);
  const bool trunc = ratio >= p.is_cap;
  const double lo_c = 1.0 - p.eps_low, hi_c = 1.0 + p.eps_high;
  const double rc = fmin(fmax(r, lo_c), hi_c);
  const double sur = fmin(r * A, rc * A);                      // Eq. 1 min(rA, clip(r)A)
  const bool act = (A > 0.0) ? (r <= hi_c) : ((A < 0.0) ? (r >= lo_c) : true);
  double kl = 0.0, dkl = 0.0;
  if (p.beta != 0.0) {                                         // k3 estimator
    const double d = lref - logp;
    const double ed = exp(d);
    kl = ed - d - 1.0;
    dkl = 1.0 - ed;
  }
  const double ell = -w * sur + p.beta * kl;                   // L = -J_HE per token
  const double dell = -w * (act ? A * r : 0.0) + p.beta * dkl;
  if (!isfinite((float)ell) || !isfinite((float)dell)) bits |= DART_STATUS_NONFINITE_LOSS;
  if (lane == 0) {
    p.lse[row] = (float)lse;
    p.logp[row] = (float)logp;
    p.H[row] = (float)H;
    p.ell[row] = (float)ell;
    p.dell[row] = (float)dell;
    p.lse2[row] = (float)lse2;
    p.aux_w[row] = (float)w;
    p.aux_kl[row] = (float)kl;
    p.aux_flags[row] = (uint8_t)((act ? 0u : 1u) | (trunc ? 2u : 0u));
    status_or(p.status, bits);
  }
}

__device__ __forceinline__ void row_epilogue(const FwdParams& p, int64_t row, Part R, uint32_t bits, bool is_bf16,
                                             int lane) {
  const int32_t y = p.target[row];
  float zy = __int_as_float(0x7fc00000);
  if (y < 0 || y >= p.V) bits |= DART_STATUS_TARGET_RANGE;
  else zy = load_logit(p, row, y, is_bf16);
  row_epilogue_z(p, row, R, bits, zy, lane);
}

// Issue the bulk copy of the producer stream's next chunk into `slot` and advance it.
__device__ __forceinline__ void issue_next(Stream& ps, uint64_t* bars, uint8_t* ring, int slot, const FwdParams& p,
                                           int64_t W, int64_t units, int lg, int64_t nvec, int lane, uint64_t pol) {
  const int nv = min(FCH_VEC, ps.vend - ps.v);
  if (lane == 0) {
    mbar_arrive_expect_tx(&bars[slot], (uint32_t)nv * 16u);
    bulk_g2s_hint(ring + (size_t)slot * FCH_BYTES, p.logits + ps.row * p.ld_bytes + (int64_t)ps.v * 16,
                  (uint32_t)nv * 16u, &bars[slot], pol);
  }
  ps.v += nv;
  if (ps.v == ps.vend) stream_next_segment(ps, W, units, lg, nvec);
}

// Hand the slot back to the copy engine right after this chunk's shared loads
// (fence_reads_before_refill orders them before the async-proxy refill) and
// refill it STAGES chunks ahead.
template <int STAGES>
__device__ __forceinline__ void release_refill(const uint4 (&x)[FVPL], uint64_t* bars, uint8_t* ring, int slot,
                                               Stream& ps, const FwdParams& p, int64_t W, int64_t units, int lg,
                                               int64_t nvec, int lane, uint64_t pol) {
  (void)x;
  fence_reads_before_refill();
  __syncwarp();
  if (ps.valid) issue_next(ps, bars, ring, slot, p, W, units, lg, nvec, lane, pol);
}

// ============================================================== K1
template <typename Tin, int WARPS, int STAGES>
__global__ void __launch_bounds__(WARPS * 32)
fwd_sweep_kernel(const FwdParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + (size_t)warp * STAGES * FCH_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)WARPS * STAGES * FCH_BYTES) + warp * STAGES;
  constexpr bool IS_BF16 = sizeof(Tin) == 2;
  constexpr int EPV = 16 / sizeof(Tin);

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();

  const int64_t W = (int64_t)gridDim.x * WARPS;
  const int64_t wid = (int64_t)blockIdx.x * WARPS + warp;
  const int lg = p.lg_nsplit;
  const int nsplit = 1 << lg;
  const int64_t units = p.T_loc << lg;
  const int64_t nvec = p.nvec;
  const float c2 = p.c2;
  const float m0 = NEG_CLAMP * c2;
  // the row's last vector is partial when V*sizeof % 16 != 0
  const int tail_elems = (int)(p.V % EPV);
  const uint32_t tail_keep = tail_elems ? ((1u << tail_elems) - 1u) : 0xffu;
  const uint64_t pol = policy_evict_first();

  Stream cs, ps;
  stream_set_unit(cs, wid, units, lg, nvec);
  ps = cs;
  // prologue: fill the ring
#pragma unroll 1
  for (int s = 0; s < STAGES; ++s) {
    if (!ps.valid) break;
    issue_next(ps, bars, ring, s, p, W, units, lg, nvec, lane, pol);
  }

  int slot = 0;
  uint32_t phase = 0;
  LaneAcc a;
  acc_reset(a, m0);
  Part rowp = {-INFINITY, 0.0, 0.0};
  uint32_t bad = 0;

#pragma unroll 1
  while (cs.valid) {
    const int64_t row = cs.row;
    const int32_t v0 = cs.v;
    const int nv = min(FCH_VEC, cs.vend - cs.v);
    const int k = cs.k;
    cs.v += nv;
    const bool seg_end = (cs.v == cs.vend);
    bool unit_end = false;
    if (seg_end) unit_end = stream_next_segment(cs, W, units, lg, nvec);
    mbar_wait(&bars[slot], phase);
    const uint8_t* sp = ring + (size_t)slot * FCH_BYTES;
    const int tail_idx = (tail_elems && (int64_t)v0 + nv == nvec) ? nv - 1 : -1;
    if (nv == FCH_VEC && tail_idx < 0) {
      uint4 x[FVPL];
#pragma unroll
      for (int kk = 0; kk < FVPL; ++kk) x[kk] = lds128(sp + (lane + 32 * kk) * 16);
      release_refill<STAGES>(x, bars, ring, slot, ps, p, W, units, lg, nvec, lane, pol);
      if (IS_BF16) chunk_bf16<true>(x, nv, lane, c2, a, bad, -1, tail_keep);
      else chunk_f32<true>(x, nv, lane, c2, a, bad, -1, tail_keep);
    } else {
      uint4 x[FVPL];
#pragma unroll
      for (int kk = 0; kk < FVPL; ++kk) {
        const int vi = lane + 32 * kk;
        x[kk] = (vi < nv) ? lds128(sp + vi * 16) : make_uint4(0u, 0u, 0u, 0u);
      }
      release_refill<STAGES>(x, bars, ring, slot, ps, p, W, units, lg, nvec, lane, pol);
      if (IS_BF16) chunk_bf16<false>(x, nv, lane, c2, a, bad, tail_idx, tail_keep);
      else chunk_f32<false>(x, nv, lane, c2, a, bad, tail_idx, tail_keep);
    }
    if (++slot == STAGES) { slot = 0; phase ^= 1u; }

    if (seg_end) {
      // --- canonical segment reduction: lanes -> one (M, S, U)
      const float sl = ((a.s[0].x + a.s[0].y) + (a.s[1].x + a.s[1].y)) + ((a.s[2].x + a.s[2].y) + (a.s[3].x + a.s[3].y));
      const float ul = ((a.u[0].x + a.u[0].y) + (a.u[1].x + a.u[1].y)) + ((a.u[2].x + a.u[2].y) + (a.u[3].x + a.u[3].y));
      const uint32_t wbad = warp_or(bad);
      Part seg;
      if (__any_sync(0xffffffffu, isnan(ul) || isnan(sl)) && !wbad) {
        seg = segment_slow<Tin>(p, row, k, lane);      // -inf logits in the segment
      } else {
        const float M = warp_max_f(a.m);
        const float dmf = a.m - M;
        const double dm = (double)dmf;
        const double f = (double)ex2(dmf);
        seg.m = (double)M;
        seg.s = warp_sum_d((double)sl * f);
        seg.u = warp_sum_d(((double)ul + (double)sl * dm) * f);
      }
      acc_reset(a, m0);
      if (nsplit == 1) {
        rowp = part_fold(rowp, seg);
      } else if (lane == 0) {
        const int64_t idx = row * KSEG + k;
        p.part_m[idx] = (float)seg.m;
        p.part_s[idx] = seg.s;
        p.part_u[idx] = seg.u;
      }
      if (unit_end) {
        const uint32_t rbits = warp_or(bad);
        bad = 0;
        if (nsplit == 1) {
          row_epilogue(p, row, rowp, rbits, IS_BF16, lane);
          rowp = {-INFINITY, 0.0, 0.0};
        } else {
          // last-arriving warp of the row folds the KSEG partials in order
          __threadfence();
          uint32_t prev = 0;
          if (lane == 0) prev = atomicAdd(&p.row_cnt[row], 1u);
          prev = __shfl_sync(0xffffffffu, prev, 0);
          if (lane == 0) status_or(p.status, rbits);
          if (prev == (uint32_t)(nsplit - 1)) {
            __threadfence();
            Part R = {-INFINITY, 0.0, 0.0};
            for (int kk = 0; kk < KSEG; ++kk) {
              if (seg_begin(nvec, kk + 1) == seg_begin(nvec, kk)) continue;
              const int64_t idx = row * KSEG + kk;
              Part q;
              q.m = (double)__ldcg(&p.part_m[idx]);
              q.s = __ldcg(&p.part_s[idx]);
              q.u = __ldcg(&p.part_u[idx]);
              R = part_fold(R, q);
            }
            row_epilogue(p, row, R, 0u, IS_BF16, lane);
          }
        }
      }
    }
  }
}

// ============================================================== LM-head combine
// fold the per-(row, vocabulary chunk) partials the tcgen05
// LM-head kernel left (dart_lmhead.cu) in chunk order, then the same row
// epilogue as the logits sweep.  One thread per row; deterministic.
__global__ void lmhead_combine_kernel(FwdParams p, LmCombineParams c) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= p.T_loc) return;
  Part R = {-INFINITY, 0.0, 0.0};
  const int64_t base = row * c.n_nc;
  for (int k = 0; k < c.n_nc; ++k) {
    Part q;
    q.m = (double)c.part_m[base + k];
    q.s = c.part_s[base + k];
    q.u = c.part_u[base + k];
    R = part_fold(R, q);
  }
  const int32_t y = p.target[row];
  uint32_t bits = 0;
  float zy = __int_as_float(0x7fc00000);
  if (y < 0 || y >= p.V) bits |= DART_STATUS_TARGET_RANGE;
  else zy = c.zy[row];
  if (!isfinite(R.m) || !isfinite(R.s) || !isfinite(R.u) || !(bits || isfinite(zy))) bits |= DART_STATUS_NONFINITE_LOGIT;
  row_epilogue_z(p, row, R, bits, zy, 0);
}

// ============================================================== K2
// One warp per local step; fixed-order per-lane sums + xor butterfly.
// Step-ratio mode (DART_RATIO_STEP): the ratio, IS weight
// and surrogate are taken on the step's sequence log-probability
// sum_t log pi(y_t) (the literal pi(a|h,s) of PAPER.md:124, 257); the per-token
// d ell / d logp_t = -w_s A r_s act_s + beta (1 - e^{d_t}) is rewritten here.
__global__ void step_reduce_kernel(StepReduceParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool step_ratio = p.ratio_level == DART_RATIO_STEP;
  for (int64_t s = w; s < p.S_loc; s += nw) {
    const int64_t sg = p.step_begin + s;
    int64_t t0 = p.step_tok_off[sg] - p.tok_begin;
    int64_t t1 = p.step_tok_off[sg + 1] - p.tok_begin;
    t0 = max(t0, (int64_t)0);
    t1 = min(t1, p.T_loc);
    const int64_t n = t1 - t0;
    if (p.no_entropy && !p.keep[sg]) {   // fused mode: masked steps carry no per-token values
      if (lane == 0) {
        p.step_ell[s] = 0.0;
        double* st = p.step_stats + s * NSTAT;
        for (int i = 0; i < NSTAT; ++i) st[i] = 0.0;
      }
      continue;
    }
    double sH = 0, sE = 0, sw = 0, sclip = 0, strunc = 0, sA = 0, sA2 = 0, skl = 0;
    double sdl = 0, sdw = 0;  // step ratio: sum(logp - logp_old), sum(logp_old - logp_roll)
    for (int64_t t = t0 + lane; t < t1; t += 32) {
      if (!p.no_entropy) sH += (double)p.H[t];
      sE += (double)p.ell[t];
      sw += (double)p.aux_w[t];
      const uint32_t f = p.aux_flags[t];
      sclip += (double)(f & 1u);
      strunc += (double)((f >> 1) & 1u);
      const double A = (double)p.tok_adv[t];
      sA += A;
      sA2 += A * A;
      skl += (double)p.aux_kl[t];
      if (step_ratio) {
        sdl += (double)p.logp[t] - (double)p.logp_old[t];
        sdw += (double)p.logp_old[t] - (double)p.logp_roll[t];
      }
    }
    sH = warp_sum_d(sH);
    sE = warp_sum_d(sE);
    sw = warp_sum_d(sw);
    sclip = warp_sum_d(sclip);
    strunc = warp_sum_d(strunc);
    sA = warp_sum_d(sA);
    sA2 = warp_sum_d(sA2);
    skl = warp_sum_d(skl);
    if (step_ratio && n > 0) {
      sdl = warp_sum_d(sdl);
      sdw = warp_sum_d(sdw);
      const double A = (double)p.tok_adv[t0];              // one trajectory per step
      const double r = exp(sdl);
      const double ratio = exp(sdw);
      const double wt = fmin(ratio, p.is_cap);
      const bool trunc = ratio >= p.is_cap;
      const double lo_c = 1.0 - p.eps_low, hi_c = 1.0 + p.eps_high;
      const double rc = fmin(fmax(r, lo_c), hi_c);
      const double sur = fmin(r * A, rc * A);
      const bool act = (A > 0.0) ? (r <= hi_c) : ((A < 0.0) ? (r >= lo_c) : true);
      const double ell_s = -wt * sur + p.beta * skl;
      const double dsur = -wt * (act ? A * r : 0.0);
      const uint8_t flags = (uint8_t)((act ? 0u : 1u) | (trunc ? 2u : 0u));
      bool bad = !isfinite(ell_s);
      for (int64_t t = t0 + lane; t < t1; t += 32) {
        double dkl = 0.0;
        if (p.beta != 0.0 && !p.exact_kl) dkl = 1.0 - exp((double)p.logp_ref[t] - (double)p.logp[t]);
        const float dl = (float)(dsur + p.beta * dkl);
        bad |= !isfinite(dl);
        p.dell[t] = dl;
        p.ell[t] = (float)(ell_s / (double)n);
        p.aux_w[t] = (float)wt;
        p.aux_flags[t] = flags;
      }
      if (__any_sync(0xffffffffu, bad) && lane == 0) status_or(p.status, DART_STATUS_NONFINITE_LOSS);
      sE = ell_s;
      sw = wt * (double)n;
      sclip = act ? 0.0 : (double)n;
      strunc = trunc ? (double)n : 0.0;
    }
    if (lane == 0) {
      if (!p.no_entropy)
        p.step_entropy[s] = n > 0 ? (float)(sH / (double)n) : __int_as_float(0x7fc00000);
      p.step_ell[s] = sE;
      double* st = p.step_stats + s * NSTAT;
      st[0] = sw; st[1] = sclip; st[2] = strunc; st[3] = sA; st[4] = sA2; st[5] = skl; st[6] = sH;
    }
  }
}

// ============================================================== launchers
template <typename Tin, int WARPS, int STAGES>
static cudaError_t launch_fwd_sweep_t(const FwdParams& p, int num_sms, cudaStream_t st) {
  const size_t smem = (size_t)WARPS * STAGES * FCH_BYTES + (size_t)WARPS * STAGES * 8;
  auto kern = fwd_sweep_kernel<Tin, WARPS, STAGES>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WARPS * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t units = p.T_loc << p.lg_nsplit;
  int64_t grid = (int64_t)num_sms * per_sm;
  const int64_t need = (units + WARPS - 1) / WARPS;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, WARPS * 32, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_fwd_sweep(const FwdParams& p, bool bf16, int num_sms, cudaStream_t st) {
  if (bf16) return launch_fwd_sweep_t<__nv_bfloat16, FWD_WARPS, FWD_STAGES>(p, num_sms, st);
  return launch_fwd_sweep_t<float, FWD_WARPS, FWD_STAGES>(p, num_sms, st);
}

cudaError_t launch_lmhead_combine(const FwdParams& p, const LmCombineParams& c, cudaStream_t st) {
  if (p.T_loc <= 0) return cudaSuccess;
  lmhead_combine_kernel<<<(unsigned)((p.T_loc + 127) / 128), 128, 0, st>>>(p, c);
  return cudaGetLastError();
}

cudaError_t launch_adv(const AdvParams& p, cudaStream_t st) {
  int64_t n = p.G;
  if (p.N_traj > n) n = p.N_traj;
  if (p.S > n) n = p.S;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) blocks = 1;
  adv_kernel<<<(unsigned)blocks, 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_tok_meta(const TokMetaParams& p, cudaStream_t st) {
  int64_t warps = p.S_loc > 0 ? p.S_loc : 1;
  int64_t blocks = (warps * 32 + 255) / 256;
  if (blocks > 8192) blocks = 8192;
  tok_meta_kernel<<<(unsigned)blocks, 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_step_reduce(const StepReduceParams& p, cudaStream_t st) {
  if (p.S_loc <= 0) return cudaSuccess;
  int64_t blocks = (p.S_loc * 32 + 255) / 256;
  if (blocks > 8192) blocks = 8192;
  step_reduce_kernel<<<(unsigned)blocks, 256, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace dart
