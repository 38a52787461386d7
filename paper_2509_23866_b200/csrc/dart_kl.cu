// dart_kl.cu -- SURVEY §8(f) NEXT #4: exact full-vocabulary KL(pi_theta || pi_ref)
// from the reference policy's logits (sm_100a).
//
// KL_t = sum_v p_v (log p_v - log q_v)  (D_KL(pi_theta || pi_ref),
// estimator unstated -- SURVEY Q10), p = softmax(z/T), q = softmax(z_ref/T).
// In log2 units x = z c2, xr = z_ref c2 (c2 = invT log2 e):
//     KL_t = ln2 (sum_v p_v (x_v - xr_v) - lse2 + lse2_ref)
//     dKL_t/dz_v = invT p_v (invT (z_v - zr_v) - Q_t),  Q_t = ln2 (lse2 - lse2_ref) + KL_t
// so each sweep streams both rows: K1k (forward: online max/sum/entropy of
// z, online max/sum of z_ref, and D = sum e (x - xr)) and K4k (gradient:
// p_v (-g + h (invT (z_v - zr_v) - Q_t)) + g [v = y]).  Ring slots hold a
// 2 KB chunk of z and the matching 2 KB of z_ref (one mbarrier transaction).
// One warp reduces one row (no split mode), so results do not depend on how
// rows are distributed.
#include "dart_common.cuh"
#include "dart_internal.h"

namespace dart {

constexpr int KV = CH_VEC / 2;      // 16-byte vectors per stream per chunk (2 KB)
constexpr int KVPL = KV / 32;       // vectors per lane per stream
constexpr float KL_LAZY = 2.0f;
constexpr int KL_FLUSH = 8;   // chunks between fp32 -> fp64 flushes (power of two)

template <typename Tin>
__device__ __forceinline__ void unpack8(const uint4& xv, float* z) {
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
__device__ __forceinline__ uint4 neg_clamp_vec() {
  if (sizeof(Tin) == 2) {
    const uint32_t w = NEG_CLAMP_BF16 | (NEG_CLAMP_BF16 << 16);
    return make_uint4(w, w, w, w);
  }
  const uint32_t w = __float_as_uint(NEG_CLAMP);
  return make_uint4(w, w, w, w);
}

// logits at positions >= keep of the row's last vector are not part of the row
template <typename Tin>
__device__ __forceinline__ void mask_tail(uint4& v, int keep) {
  uint32_t* w = reinterpret_cast<uint32_t*>(&v);
  if (sizeof(Tin) == 2) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (2 * j >= keep) w[j] = (w[j] & 0xffff0000u) | NEG_CLAMP_BF16;
      if (2 * j + 1 >= keep) w[j] = (w[j] & 0x0000ffffu) | (NEG_CLAMP_BF16 << 16);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j >= keep) w[j] = __float_as_uint(NEG_CLAMP);
  }
}

template <typename Tin>
__device__ __forceinline__ void chunk_max(const uint4 (&x)[KVPL], float& cm) {
  if (sizeof(Tin) == 2) {
    uint32_t mx = 0xff80ff80u;
#pragma unroll
    for (int q = 0; q < KVPL; ++q) {
      mx = bmax2_nan(mx, x[q].x);
      mx = bmax2_nan(mx, x[q].y);
      mx = bmax2_nan(mx, x[q].z);
      mx = bmax2_nan(mx, x[q].w);
    }
    cm = fmax_nan(bf16lo(mx), bf16hi(mx));
  } else {
    cm = -INFINITY;
#pragma unroll
    for (int q = 0; q < KVPL; ++q) {
      cm = fmax_nan(cm, __uint_as_float(x[q].x));
      cm = fmax_nan(cm, __uint_as_float(x[q].y));
      cm = fmax_nan(cm, __uint_as_float(x[q].z));
      cm = fmax_nan(cm, __uint_as_float(x[q].w));
    }
  }
}

template <typename Tin>
__device__ __forceinline__ void unpack_clamped(const uint4& xv, float* z) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(&xv);
  if (sizeof(Tin) == 2) {
    const uint32_t cl = NEG_CLAMP_BF16 | (NEG_CLAMP_BF16 << 16);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t c = bmax2(w[j], cl);   // packed clamp of -inf (NaN -> clamp; flagged separately)
      z[2 * j] = bf16lo(c);
      z[2 * j + 1] = bf16hi(c);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) z[j] = fmaxf(__uint_as_float(w[j]), NEG_CLAMP);
  }
}

template <typename Tin>
__device__ __forceinline__ float logit_at(const uint8_t* row, int64_t y) {
  if (sizeof(Tin) == 2) return __uint_as_float(((uint32_t)(*reinterpret_cast<const uint16_t*>(row + 2 * y))) << 16);
  return *reinterpret_cast<const float*>(row + 4 * y);
}

// per-row epilogue of the exact-KL forward (token-level ratio; the step-ratio
// mode re-derives dell in the step reduce)
__device__ void kl_row_epilogue(const FwdParams& p, int64_t row, double M, double S, double U, double Mr, double Sr,
                                double Dd, uint32_t bits, bool is_bf16, int lane) {
  const int32_t y = p.target[row];
  const double lo = p.logp_old[row], lr = p.logp_roll[row];
  const double A = p.tok_adv[row];
  float zy = __int_as_float(0x7fc00000);
  if (y < 0 || y >= p.V) bits |= DART_STATUS_TARGET_RANGE;
  else zy = is_bf16 ? logit_at<__nv_bfloat16>(p.logits + row * p.ld_bytes, y) : logit_at<float>(p.logits + row * p.ld_bytes, y);
  if (!isfinite(lo) || !isfinite(lr)) bits |= DART_STATUS_NONFINITE_LOGP;
  if (zy == -INFINITY) bits |= DART_STATUS_TARGET_NEGINF;
  if (M <= (double)clamp_max0(p.c2)) bits |= DART_STATUS_ROW_ALL_NEGINF;
  const double L2s = log2(S), L2r = log2(Sr);
  const double lse2 = M + L2s, lse2r = Mr + L2r;
  double H = LN2_D * (L2s - U / S);
  if (H < 0.0) H = 0.0;
  const double logp = ((double)zy * (double)p.c2 - M - L2s) * LN2_D;
  double kl = LN2_D * (Dd / S - lse2 + lse2r);
  if (kl < 0.0) kl = 0.0;   // Gibbs: rounding only
  const double Q = LN2_D * (lse2 - lse2r) + kl;
  const double r = exp(logp - lo);
  const double ratio = exp(lo - lr);
  const double w = fmin(ratio, p.is_cap);
  const bool trunc = ratio >= p.is_cap;
  const double lo_c = 1.0 - p.eps_low, hi_c = 1.0 + p.eps_high;
  const double rc = fmin(fmax(r, lo_c), hi_c);
  const double sur = fmin(r * A, rc * A);
  const bool act = (A > 0.0) ? (r <= hi_c) : ((A < 0.0) ? (r >= lo_c) : true);
  const double ell = -w * sur + p.beta * kl;
  const double dell = -w * (act ? A * r : 0.0);   // the KL gradient is per element (bwd)
  if (!isfinite((float)ell) || !isfinite((float)dell)) bits |= DART_STATUS_NONFINITE_LOSS;
  if (lane == 0) {
    p.lse[row] = (float)(lse2 * LN2_D);
    p.logp[row] = (float)logp;
    p.H[row] = (float)H;
    p.ell[row] = (float)ell;
    p.dell[row] = (float)dell;
    p.lse2[row] = (float)lse2;
    p.aux_w[row] = (float)w;
    p.aux_kl[row] = (float)kl;
    p.aux_flags[row] = (uint8_t)((act ? 0u : 1u) | (trunc ? 2u : 0u));
    p.klq[row] = (float)Q;
    status_or(p.status, bits);
  }
}

// ============================================================== K1k
template <typename Tin, int WARPS, int STAGES>
__global__ void __launch_bounds__(WARPS * 32)
fwd_kl_kernel(const FwdParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int EPV = 16 / sizeof(Tin);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + (size_t)warp * STAGES * CH_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)WARPS * STAGES * CH_BYTES) + warp * STAGES;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const int64_t W = (int64_t)gridDim.x * WARPS;
  const int64_t wid = (int64_t)blockIdx.x * WARPS + warp;
  const int64_t nvec = p.nvec;
  const int64_t nchk = (nvec + KV - 1) / KV;
  const float c2 = p.c2;
  const int tail_elems = (int)(p.V % EPV);
  const uint64_t pol = policy_evict_first();

  // chunk stream of this warp: rows wid, wid+W, ...; chunks c = 0..nchk-1
  int64_t prow = wid, pc = 0;   // producer cursor
  auto issue = [&](int slot) {
    const int64_t v0 = pc * KV;
    const uint32_t nv = (uint32_t)min((int64_t)KV, nvec - v0);
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars[slot], 2u * nv * 16u);
      uint8_t* dst = ring + (size_t)slot * CH_BYTES;
      bulk_g2s_hint(dst, p.logits + prow * p.ld_bytes + v0 * 16, nv * 16u, &bars[slot], pol);
      bulk_g2s_hint(dst + KV * 16, p.ref_logits + prow * p.ld_ref_bytes + v0 * 16, nv * 16u, &bars[slot], pol);
    }
    if (++pc == nchk) { pc = 0; prow += W; }
  };
#pragma unroll 1
  for (int s = 0; s < STAGES; ++s) {
    if (prow >= p.T_loc) break;
    issue(s);
  }
  int slot = 0;
  uint32_t phase = 0;
#pragma unroll 1
  for (int64_t row = wid; row < p.T_loc; row += W) {
    // running maxima start at NEG_CLAMP * c2 rounded toward zero (dart_common.cuh):
    // lanes that only see NEG_CLAMP padding (rows of fewer than 32 vectors)
    float m = clamp_max0(c2), mr = clamp_max0(c2);
    float2 s[4], u[4], D[4], sr[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) s[j] = u[j] = D[j] = sr[j] = make_float2(0.f, 0.f);
    // fp64 per-lane accumulators in the same shift frame: the fp32 ones are
    // flushed into them every KL_FLUSH chunks (bounded fp32 accumulation length)
    double Sd = 0.0, Ud = 0.0, Dd_ = 0.0, Srd = 0.0;
    uint32_t bad = 0;
#pragma unroll 1
    for (int64_t c = 0; c < nchk; ++c) {
      const int64_t v0 = c * KV;
      const int nv = (int)min((int64_t)KV, nvec - v0);
      mbar_wait(&bars[slot], phase);
      const uint8_t* sp = ring + (size_t)slot * CH_BYTES;
      uint4 xz[KVPL], xr[KVPL];
#pragma unroll
      for (int q = 0; q < KVPL; ++q) {
        const int vi = lane + 32 * q;
        xz[q] = (vi < nv) ? lds128(sp + vi * 16) : make_uint4(0u, 0u, 0u, 0u);
        xr[q] = (vi < nv) ? lds128(sp + KV * 16 + vi * 16) : make_uint4(0u, 0u, 0u, 0u);
      }
      fence_reads_before_refill();
      __syncwarp();
      if (prow < p.T_loc) issue(slot);
      if (++slot == STAGES) { slot = 0; phase ^= 1u; }
      // sanitize: vectors past nv and logits past V become NEG_CLAMP (exp -> 0)
#pragma unroll
      for (int q = 0; q < KVPL; ++q) {
        const int vi = lane + 32 * q;
        if (vi >= nv) {
          xz[q] = xr[q] = neg_clamp_vec<Tin>();
        } else if (tail_elems && v0 + vi == nvec - 1) {
          mask_tail<Tin>(xz[q], tail_elems);
          mask_tail<Tin>(xr[q], tail_elems);
        }
      }
      float cm, cmr;
      chunk_max<Tin>(xz, cm);
      chunk_max<Tin>(xr, cmr);
      if (!(cm < INFINITY) || !(cmr < INFINITY)) bad |= DART_STATUS_NONFINITE_LOGIT;
      const float cms = fmaxf(cm, NEG_CLAMP) * c2, cmrs = fmaxf(cmr, NEG_CLAMP) * c2;
      if (__any_sync(0xffffffffu, cms > m + KL_LAZY)) {
        const float mn = (cms > m + KL_LAZY) ? cms : m;
        const float dm = m - mn, sc = ex2(dm);
        const float2 dm2 = make_float2(dm, dm), sc2 = make_float2(sc, sc);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          u[j] = __fmul2_rn(__ffma2_rn(s[j], dm2, u[j]), sc2);
          s[j] = __fmul2_rn(s[j], sc2);
          D[j] = __fmul2_rn(D[j], sc2);
        }
        Ud = (Ud + Sd * (double)dm) * (double)sc;
        Sd *= (double)sc;
        Dd_ *= (double)sc;
        m = mn;
      }
      if (__any_sync(0xffffffffu, cmrs > mr + KL_LAZY)) {
        const float mn = (cmrs > mr + KL_LAZY) ? cmrs : mr;
        const float sc = ex2(mr - mn);
        const float2 sc2 = make_float2(sc, sc);
#pragma unroll
        for (int j = 0; j < 4; ++j) sr[j] = __fmul2_rn(sr[j], sc2);
        Srd *= (double)sc;
        mr = mn;
      }
      const float2 cc = make_float2(c2, c2), nm = make_float2(-m, -m), nmr = make_float2(-mr, -mr);
#pragma unroll
      for (int q = 0; q < KVPL; ++q) {
        float zz[8], zq[8];
        unpack_clamped<Tin>(xz[q], zz);   // -inf -> NEG_CLAMP: 0 * -inf would poison u and D
        unpack_clamped<Tin>(xr[q], zq);
#pragma unroll
        for (int e = 0; e < EPV; e += 2) {
          const int j = (e / 2) & 3;
          const float2 z2 = make_float2(zz[e], zz[e + 1]);
          const float2 r2 = make_float2(zq[e], zq[e + 1]);
          const float2 d = __ffma2_rn(z2, cc, nm);
          const float2 ee = make_float2(ex2(d.x), ex2(d.y));
          s[j] = __fadd2_rn(s[j], ee);
          u[j] = __ffma2_rn(ee, d, u[j]);
          const float2 dr = __ffma2_rn(r2, cc, nmr);
          sr[j] = __fadd2_rn(sr[j], make_float2(ex2(dr.x), ex2(dr.y)));
          const float2 df = __fmul2_rn(__fadd2_rn(z2, make_float2(-r2.x, -r2.y)), cc);   // x - xr
          D[j] = __ffma2_rn(ee, df, D[j]);
        }
      }
      if ((c & (KL_FLUSH - 1)) == KL_FLUSH - 1 || c == nchk - 1) {   // flush fp32 -> fp64 (fixed points)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          Sd += (double)s[j].x + (double)s[j].y;
          Ud += (double)u[j].x + (double)u[j].y;
          Dd_ += (double)D[j].x + (double)D[j].y;
          Srd += (double)sr[j].x + (double)sr[j].y;
          s[j] = u[j] = D[j] = sr[j] = make_float2(0.f, 0.f);
        }
      }
    }
    // ---- row reduction (fixed lane order) and epilogue
    const float M = warp_max_f(m), Mr = warp_max_f(mr);
    const double f = (double)ex2(m - M), fr = (double)ex2(mr - Mr);
    const double dmf = (double)(m - M);
    const double S = warp_sum_d(Sd * f);
    const double U = warp_sum_d((Ud + Sd * dmf) * f);
    const double Dd = warp_sum_d(Dd_ * f);
    const double Sr = warp_sum_d(Srd * fr);
    const uint32_t rbits = warp_or(bad);
    kl_row_epilogue(p, row, (double)M, S, U, (double)Mr, Sr, Dd, rbits, sizeof(Tin) == 2, lane);
  }
}

// ============================================================== K4ak (row records)
__global__ void rowrec_kl_kernel(RowRecParams p) {
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < p.T_loc; t += nthreads) {
    const double cs = p.step_scale[p.tok_step[t]];
    const float g = (float)(cs * (double)p.dell[t] * p.invT);
    const double h = p.beta * cs * p.invT;
    int32_t y = p.target[t];
    float zy = 0.f, zry = 0.f;
    if (y >= 0 && y < p.V) {
      zy = p.is_bf16 ? logit_at<__nv_bfloat16>(p.logits + t * p.ld_bytes, y) : logit_at<float>(p.logits + t * p.ld_bytes, y);
      zry = p.is_bf16 ? logit_at<__nv_bfloat16>(p.ref_logits + t * p.ld_ref_bytes, y)
                      : logit_at<float>(p.ref_logits + t * p.ld_ref_bytes, y);
    } else {
      y = -1;
    }
    float4* r = reinterpret_cast<float4*>(p.rec) + 2 * t;
    r[0] = make_float4(g, -p.lse2[t], __int_as_float(y), zy);
    r[1] = make_float4(zry, (float)(h * p.invT), (float)(-(double)g - h * (double)p.klq[t]), 0.f);
  }
}

// ============================================================== K4k
struct KCur {
  int64_t j, jend, s, t, tend;
  int32_t c;
  bool kept, valid;
};

__device__ __forceinline__ void kcur_seek(KCur& o, const BwdParams& p, int64_t j) {
  o.j = j;
  o.valid = j < o.jend;
  if (!o.valid) return;
  const int64_t s = upper_bound_i64(p.step_chunk, 0, p.S_loc + 1, j) - 1;
  o.s = s;
  const int64_t sg = p.step_begin + s;
  const int64_t off = j - p.step_chunk[s];
  o.t = p.step_tok_off[sg] - p.tok_begin + off / p.nch;
  o.tend = p.step_tok_off[sg + 1] - p.tok_begin;
  o.c = (int32_t)(off % p.nch);
  o.kept = p.keep[sg] != 0;
}

__device__ __forceinline__ void kcur_advance(KCur& o, const BwdParams& p, int stride) {
  o.j += stride;
  if (o.j >= o.jend) { o.valid = false; return; }
  o.c += stride;
  while (o.c >= p.nch) { o.c -= (int32_t)p.nch; ++o.t; }
  if (o.t >= o.tend) kcur_seek(o, p, o.j);
}

__device__ __forceinline__ void kcur_to_kept(KCur& o, const BwdParams& p, int stride) {
  while (o.valid && !o.kept) {
    const int64_t nxt = p.step_chunk[o.s + 1];
    const int64_t k = (nxt - o.j + stride - 1) / stride;
    kcur_seek(o, p, o.j + k * stride);
  }
}

__device__ __forceinline__ int64_t kl_ordinal_at_cost(const BwdParams& p, int64_t x) {
  const int64_t total = p.step_cost[p.S_loc];
  if (x >= total) return p.step_chunk[p.S_loc];
  const int64_t s = upper_bound_i64(p.step_cost, 0, p.S_loc + 1, x) - 1;
  const int uc = p.keep[p.step_begin + s] ? 3 : 1;   // kept: read z + z_ref + write; masked: write
  const int64_t off = (x - p.step_cost[s] + uc - 1) / uc;
  const int64_t n = p.step_chunk[s + 1] - p.step_chunk[s];
  return off >= n ? p.step_chunk[s + 1] : p.step_chunk[s] + off;
}

template <typename Tin, typename Tout, int WARPS, int STAGES>
__global__ void __launch_bounds__(WARPS * 32, 1)
bwd_kl_kernel(const BwdParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int EPV = 16 / sizeof(Tin);
  constexpr bool OUT_BF16 = sizeof(Tout) == 2;
  constexpr int64_t OUTV = EPV * (int64_t)sizeof(Tout);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + (size_t)warp * STAGES * CH_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)WARPS * STAGES * CH_BYTES) + warp * STAGES;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const int64_t total = p.step_cost[p.S_loc];
  const int64_t nb = gridDim.x;
  const int64_t J0 = kl_ordinal_at_cost(p, (total * (int64_t)blockIdx.x) / nb);
  const int64_t J1 = kl_ordinal_at_cost(p, (total * ((int64_t)blockIdx.x + 1)) / nb);
  const int tail_elems = (int)(p.V % EPV);
  const float c2 = p.c2;
  const uint64_t pol = policy_evict_first();
  const float4* rec = reinterpret_cast<const float4*>(p.rec);
  const int64_t nvec = p.nvec;

  KCur cc;
  cc.jend = J1;
  kcur_seek(cc, p, J0 + warp);
  KCur pc = cc;
  kcur_to_kept(pc, p, WARPS);
  auto issue = [&](int slot) {
    const int64_t v0 = (int64_t)pc.c * KV;
    const uint32_t nv = (uint32_t)min((int64_t)KV, nvec - v0);
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars[slot], 2u * nv * 16u);
      uint8_t* dst = ring + (size_t)slot * CH_BYTES;
      bulk_g2s_hint(dst, p.logits + pc.t * p.ld_bytes + v0 * 16, nv * 16u, &bars[slot], pol);
      bulk_g2s_hint(dst + KV * 16, p.ref_logits + pc.t * p.ld_ref_bytes + v0 * 16, nv * 16u, &bars[slot], pol);
    }
    kcur_advance(pc, p, WARPS);
    kcur_to_kept(pc, p, WARPS);
  };
#pragma unroll 1
  for (int s = 0; s < STAGES; ++s) {
    if (!pc.valid) break;
    issue(s);
  }
  int slot = 0;
  uint32_t phase = 0;
  int64_t cur_t = -1;
  float4 r0 = make_float4(0, 0, 0, 0), r1 = make_float4(0, 0, 0, 0);
#pragma unroll 1
  while (cc.valid) {
    const int64_t t = cc.t;
    const int64_t v0 = (int64_t)cc.c * KV;
    const int nv = (int)min((int64_t)KV, nvec - v0);
    uint8_t* orow = p.dlogits + t * p.ldg_bytes;
    if (cc.kept) {
      if (t != cur_t) {
        cur_t = t;
        r0 = rec[2 * t];
        r1 = rec[2 * t + 1];
      }
      const float g = r0.x, nl2 = r0.y, zy = r0.w, zry = r1.x, a = r1.y, b = r1.z;
      const int32_t y = __float_as_int(r0.z);
      mbar_wait(&bars[slot], phase);
      const uint8_t* sp = ring + (size_t)slot * CH_BYTES;
      uint4 xz[KVPL], xr[KVPL];
#pragma unroll
      for (int q = 0; q < KVPL; ++q) {
        const int vi = lane + 32 * q;
        xz[q] = (vi < nv) ? lds128(sp + vi * 16) : make_uint4(0u, 0u, 0u, 0u);
        xr[q] = (vi < nv) ? lds128(sp + KV * 16 + vi * 16) : make_uint4(0u, 0u, 0u, 0u);
      }
      fence_reads_before_refill();
      __syncwarp();
      if (pc.valid) issue(slot);
      if (++slot == STAGES) { slot = 0; phase ^= 1u; }
      const float2 cc2 = make_float2(c2, c2), nl = make_float2(nl2, nl2), aa = make_float2(a, a), bb = make_float2(b, b);
#pragma unroll
      for (int q = 0; q < KVPL; ++q) {
        const int vi = lane + 32 * q;
        if (vi < nv) {
          const int64_t gv = v0 + vi;
          float zz[8], zq[8], o[8];
          unpack8<Tin>(xz[q], zz);
          unpack8<Tin>(xr[q], zq);
#pragma unroll
          for (int e = 0; e < EPV; e += 2) {
            const float2 z2 = make_float2(zz[e], zz[e + 1]);
            const float2 d = __ffma2_rn(z2, cc2, nl);
            const float2 pr = make_float2(ex2(d.x), ex2(d.y));
            const float2 df = __fadd2_rn(z2, make_float2(-zq[e], -zq[e + 1]));       // z - z_ref
            const float2 tt = __ffma2_rn(aa, df, bb);   // -g + h (invT (z - zr) - Q)
            const float2 dz = __fmul2_rn(pr, tt);
            // p = 0 (z = -inf) -> 0 even when z - zr is not finite
            o[e] = (pr.x == 0.f) ? 0.f : dz.x;
            o[e + 1] = (pr.y == 0.f) ? 0.f : dz.y;
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
              if (OUT_BF16) reinterpret_cast<__nv_bfloat16*>(orow)[gv * EPV + e] = __float2bfloat16_rn(o[e]);
              else reinterpret_cast<float*>(orow)[gv * EPV + e] = o[e];
            }
          }
        }
      }
      if (y >= 0) {   // target: p_y t_y + g
        const int64_t yv = y / EPV;
        if (yv >= v0 && yv < v0 + nv && lane == (int)((yv - v0) & 31)) {
          const float py = ex2(fmaf(zy, c2, nl2));
          const float ty = fmaf(a, zy - zry, b);
          const float dzy = fmaf(py, ty, g);
          if (OUT_BF16) reinterpret_cast<__nv_bfloat16*>(orow)[y] = __float2bfloat16_rn(dzy);
          else reinterpret_cast<float*>(orow)[y] = dzy;
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < KVPL; ++q) {
        const int vi = lane + 32 * q;
        if (vi < nv) {
          const int64_t gv = v0 + vi;
          const int nvalid = (tail_elems && gv == nvec - 1) ? tail_elems : EPV;
          uint8_t* dst = orow + gv * OUTV;
          if (nvalid == EPV) {
            if (OUT_BF16 && EPV == 8) stg128_cs(dst, make_uint4(0u, 0u, 0u, 0u));
            else if (OUT_BF16) *reinterpret_cast<uint2*>(dst) = make_uint2(0u, 0u);
            else
              for (int e = 0; e < EPV; e += 4) stg128_cs(dst + 4 * e, make_uint4(0u, 0u, 0u, 0u));
          } else {
            for (int e = 0; e < nvalid; ++e) {
              if (OUT_BF16) reinterpret_cast<__nv_bfloat16*>(orow)[gv * EPV + e] = __float2bfloat16_rn(0.f);
              else reinterpret_cast<float*>(orow)[gv * EPV + e] = 0.f;
            }
          }
        }
      }
    }
    kcur_advance(cc, p, WARPS);
  }
}

// ============================================================== launchers
template <typename Tin>
static cudaError_t launch_fwd_kl_t(const FwdParams& p, int num_sms, cudaStream_t st) {
  constexpr int WARPS = FWD_WARPS, STAGES = FWD_STAGES;
  const size_t smem = (size_t)WARPS * STAGES * CH_BYTES + (size_t)WARPS * STAGES * 8;
  auto kern = fwd_kl_kernel<Tin, WARPS, STAGES>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WARPS * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)num_sms * per_sm;
  const int64_t need = (p.T_loc + WARPS - 1) / WARPS;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, WARPS * 32, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_fwd_kl(const FwdParams& p, bool bf16, int num_sms, cudaStream_t st) {
  return bf16 ? launch_fwd_kl_t<__nv_bfloat16>(p, num_sms, st) : launch_fwd_kl_t<float>(p, num_sms, st);
}

cudaError_t launch_rowrec_kl(const RowRecParams& p, cudaStream_t st) {
  if (p.T_loc <= 0) return cudaSuccess;
  int64_t blocks = (p.T_loc + 255) / 256;
  if (blocks > 8192) blocks = 8192;
  rowrec_kl_kernel<<<(unsigned)blocks, 256, 0, st>>>(p);
  return cudaGetLastError();
}

template <typename Tin, typename Tout>
static cudaError_t launch_bwd_kl_t(const BwdParams& p, int num_sms, cudaStream_t st) {
  constexpr int WARPS = BWD_WARPS, STAGES = BWD_STAGES;
  const size_t smem = (size_t)WARPS * STAGES * CH_BYTES + (size_t)WARPS * STAGES * 8;
  auto kern = bwd_kl_kernel<Tin, Tout, WARPS, STAGES>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WARPS * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  kern<<<(unsigned)(num_sms * per_sm), WARPS * 32, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_bwd_kl(const BwdParams& p, bool in_bf16, bool out_bf16, int num_sms, cudaStream_t st) {
  if (in_bf16 && out_bf16) return launch_bwd_kl_t<__nv_bfloat16, __nv_bfloat16>(p, num_sms, st);
  if (in_bf16) return launch_bwd_kl_t<__nv_bfloat16, float>(p, num_sms, st);
  if (out_bf16) return launch_bwd_kl_t<float, __nv_bfloat16>(p, num_sms, st);
  return launch_bwd_kl_t<float, float>(p, num_sms, st);
}

}  // namespace dart
