// dart_bwd.cu -- backward half of the DART loss pass (sm_100a).
//
//   K6  bwd_prep_kernel  one CTA, fixed order over the local steps: per-step
//                        loss weight c_s (normaliser of PAPER.md:255, SURVEY
//                        Q11), the local loss partial sum_{kept s} c_s sum ell
//                        and statistics (fp64), and the prefix of per-step
//                        chunk costs that balances the sweep across warps.
//   K4a rowrec_kernel    per local row: {g_t = c_s dell_t invT, -lse2_t, y_t, z_{t,y}}.
//   K4  bwd_sweep        THE SECOND HOT LOOP: for rows of kept steps, re-read
//                        the logits (bulk copies into a per-warp ring) and
//                        write dL/dz_v = g_t (delta_{v,y} - p_v) rounded to
//                        bf16 (RNE); rows of masked steps are written as
//                        zeros without being read (the
//                        indicator removes them from the objective).
#include "dart_common.cuh"
#include "dart_internal.h"

#ifndef DART_BWD_STYLE
#define DART_BWD_STYLE 1
#endif

namespace dart {

// ============================================================== K6
constexpr int NV = 11;  // dart_stats fields

__global__ void __launch_bounds__(1024) bwd_prep_kernel(BwdPrepParams p) {
  __shared__ double red[32][NV];
  __shared__ long long wsum[32];
  __shared__ long long s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const dart_norm* nrm = reinterpret_cast<const dart_norm*>(p.norm);
  const double inv_norm = nrm->inv_norm;
  // per-step 1/n_s factor of the step-mean modes; in step-ratio mode the loss
  // term is already per step (ell_s), so no 1/n_s in any mode
  const bool step_mode = p.ratio_level != DART_RATIO_STEP &&
                         (p.norm_mode == DART_NORM_STEP_MEAN_KEPT || p.norm_mode == DART_NORM_STEP_MEAN_ALL);
  double tot[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) tot[i] = 0.0;  // meaningful in thread 0 only
  __shared__ long long wsum2[32];
  __shared__ long long s_carry2;
  if (tid == 0) { s_carry = 0; p.step_cost[0] = 0; s_carry2 = 0; p.step_chunk[0] = 0; }
  __syncthreads();
  for (int64_t base = 0; base < p.S_loc; base += blockDim.x) {
    const int64_t s = base + tid;
    double v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = 0.0;
    long long cost = 0, nchunks = 0;
    if (s < p.S_loc) {
      const int64_t sg = p.step_begin + s;
      const int64_t n = p.step_tok_off[sg + 1] - p.step_tok_off[sg];
      const bool kept = p.keep[sg] != 0;
      double c = 0.0;
      if (kept) c = step_mode ? inv_norm / (double)n : inv_norm;
      p.step_scale[s] = c;
      cost = (long long)n * p.nch * (kept ? p.kept_cost : (p.zero_fill ? 1 : 0));
      nchunks = (kept || p.zero_fill) ? (long long)n * p.nch : 0;
      const double* st = p.step_stats + s * NSTAT;
      v[1] = (double)n;          // n_tok
      if (!p.no_stats) v[9] = st[6];   // sum_H (all tokens)
      if (kept && !p.no_stats) {
        v[0] = c * p.step_ell[s];  // loss partial
        v[2] = (double)n;
        v[3] = 1.0;
        v[4] = st[1];  // clip
        v[5] = st[2];  // trunc
        v[6] = st[0];  // w
        v[7] = st[3];  // adv
        v[8] = st[4];  // adv^2
        v[10] = st[5]; // kl
      }
    }
    // --- inclusive block scan of cost
    long long x = cost, x2 = nchunks;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, o);
      const long long y2 = __shfl_up_sync(0xffffffffu, x2, o);
      if (lane >= o) { x += y; x2 += y2; }
    }
    if (lane == 31) { wsum[warp] = x; wsum2[warp] = x2; }
    // --- fixed-order reduction of v
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = warp_sum_d(v[i]);
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < NV; ++i) red[warp][i] = v[i];
    }
    __syncthreads();
    if (warp == 0) {
      long long w = (lane < (int)(blockDim.x >> 5)) ? wsum[lane] : 0;
      long long w2 = (lane < (int)(blockDim.x >> 5)) ? wsum2[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, w, o);
        const long long y2 = __shfl_up_sync(0xffffffffu, w2, o);
        if (lane >= o) { w += y; w2 += y2; }
      }
      wsum[lane] = w;  // inclusive prefix of warp totals
      wsum2[lane] = w2;
    }
    __syncthreads();
    const long long before = s_carry + (warp > 0 ? wsum[warp - 1] : 0);
    const long long before2 = s_carry2 + (warp > 0 ? wsum2[warp - 1] : 0);
    if (s < p.S_loc) {
      p.step_cost[s + 1] = before + x;
      p.step_chunk[s + 1] = before2 + x2;
    }
    if (tid == 0) {
      const int nw = blockDim.x >> 5;
      for (int w = 0; w < nw; ++w)
#pragma unroll
        for (int i = 0; i < NV; ++i) tot[i] += red[w][i];
    }
    __syncthreads();
    if (tid == 0) {
      s_carry += wsum[(blockDim.x >> 5) - 1];
      s_carry2 += wsum2[(blockDim.x >> 5) - 1];
    }
    __syncthreads();
  }
  if (tid == 0 && !p.no_stats) {
    dart_stats* o = reinterpret_cast<dart_stats*>(p.stats);
    o->loss = tot[0];
    o->n_tok = tot[1];
    o->n_kept_tok = tot[2];
    o->n_kept_step = tot[3];
    o->sum_clip = tot[4];
    o->sum_trunc = tot[5];
    o->sum_w = tot[6];
    o->sum_adv = tot[7];
    o->sum_adv2 = tot[8];
    o->sum_H = tot[9];
    o->sum_kl = tot[10];
  }
}

// ============================================================== K4a
// Per local row: the 16-byte record the sweep needs -- g_t = c_s dell_t invT,
// -lse2_t, y_t and z_{t,y} -- so a warp fetches one LDG.128 per row.
__global__ void rowrec_kernel(RowRecParams p) {
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < p.T_loc; t += nthreads) {
    const float g = (float)(p.step_scale[p.tok_step[t]] * (double)p.dell[t] * p.invT);
    int32_t y = p.target[t];
    float zy = 0.f;
    if (y >= 0 && y < p.V) {
      const uint8_t* rp = p.logits + t * p.ld_bytes;
      zy = p.is_bf16 ? __uint_as_float(((uint32_t)(*reinterpret_cast<const uint16_t*>(rp + 2 * (int64_t)y))) << 16)
                     : *reinterpret_cast<const float*>(rp + 4 * (int64_t)y);
    } else {
      y = -1;
    }
    int4 r;
    r.x = __float_as_int(g);
    r.y = __float_as_int(-p.lse2[t]);
    r.z = y;
    r.w = __float_as_int(zy);
    reinterpret_cast<int4*>(p.rec)[t] = r;
  }
}

// ============================================================== K4
// Work split: each CTA owns a contiguous, cost-balanced range of chunks
// (kept-step chunk = 2: read + write; masked = 1: write only, or absent when
// zero_fill is off), and its warps interleave over it (warp w takes chunks
// w, w+WARPS, ...).  Every SM thus streams ONE contiguous read region and ONE
// write region at a time -- far fewer concurrent DRAM streams than a
// warp-per-range split -- while still running WARPS independent rings.
constexpr int BVPL = BCH_VEC / 32;   // 16-byte vectors per lane per bwd chunk
struct OCur {
  int64_t j, jend;  // chunk ordinal (in the local chunk sequence) and the warp's end
  int64_t s;        // local step
  int64_t t, tend;  // local row, end row of the step
  int32_t c;        // chunk within the row
  bool kept, valid;
};

__device__ __forceinline__ void ocur_seek(OCur& o, const BwdParams& p, int64_t j) {
  o.j = j;
  o.valid = j < o.jend;
  if (!o.valid) return;
  // last s with step_chunk[s] <= j (empty steps skipped automatically)
  const int64_t s = upper_bound_i64(p.step_chunk, 0, p.S_loc + 1, j) - 1;
  o.s = s;
  const int64_t sg = p.step_begin + s;
  const int64_t off = j - p.step_chunk[s];
  const int64_t t0 = p.step_tok_off[sg] - p.tok_begin;
  o.tend = p.step_tok_off[sg + 1] - p.tok_begin;
  o.t = t0 + off / p.nch;
  o.c = (int32_t)(off % p.nch);
  o.kept = p.keep[sg] != 0;
}

__device__ __forceinline__ void ocur_advance(OCur& o, const BwdParams& p, int stride) {
  o.j += stride;
  if (o.j >= o.jend) { o.valid = false; return; }
  o.c += stride;
  while (o.c >= p.nch) { o.c -= (int32_t)p.nch; ++o.t; }
  if (o.t >= o.tend) ocur_seek(o, p, o.j);
}

// producer: next chunk of a kept step (masked steps are jumped over whole)
__device__ __forceinline__ void ocur_to_kept(OCur& o, const BwdParams& p, int stride) {
  while (o.valid && !o.kept) {
    const int64_t nxt = p.step_chunk[o.s + 1];
    const int64_t k = (nxt - o.j + stride - 1) / stride;
    ocur_seek(o, p, o.j + k * stride);
  }
}

// first chunk ordinal whose start cost is >= x
__device__ __forceinline__ int64_t ordinal_at_cost(const BwdParams& p, int64_t x) {
  const int64_t total = p.step_cost[p.S_loc];
  if (x >= total) return p.step_chunk[p.S_loc];
  const int64_t s = upper_bound_i64(p.step_cost, 0, p.S_loc + 1, x) - 1;
  const int uc = p.keep[p.step_begin + s] ? 2 : 1;
  const int64_t off = (x - p.step_cost[s] + uc - 1) / uc;
  const int64_t n = p.step_chunk[s + 1] - p.step_chunk[s];
  return off >= n ? p.step_chunk[s + 1] : p.step_chunk[s] + off;
}

__device__ __forceinline__ void store_vals_bf16(uint8_t* dst, const float* v, int nvalid, int EPV) {
  if (nvalid == 8 && EPV == 8) {
    uint4 o;
    o.x = pack_bf16x2(v[0], v[1]);
    o.y = pack_bf16x2(v[2], v[3]);
    o.z = pack_bf16x2(v[4], v[5]);
    o.w = pack_bf16x2(v[6], v[7]);
    stg128_cs(dst, o);
  } else if (nvalid == 4 && EPV == 4) {
    uint2 o;
    o.x = pack_bf16x2(v[0], v[1]);
    o.y = pack_bf16x2(v[2], v[3]);
    *reinterpret_cast<uint2*>(dst) = o;
  } else {
    for (int e = 0; e < nvalid; ++e) reinterpret_cast<__nv_bfloat16*>(dst)[e] = __float2bfloat16_rn(v[e]);
  }
}

__device__ __forceinline__ void store_vals_f32(uint8_t* dst, const float* v, int nvalid, int EPV) {
  if (nvalid == EPV) {
    for (int e = 0; e < EPV; e += 4)
      stg128_cs(dst + 4 * e, make_uint4(__float_as_uint(v[e]), __float_as_uint(v[e + 1]), __float_as_uint(v[e + 2]),
                                        __float_as_uint(v[e + 3])));
  } else {
    for (int e = 0; e < nvalid; ++e) reinterpret_cast<float*>(dst)[e] = v[e];
  }
}

// dz for the EPV logits of one 16-byte input vector: -g * 2^(z c2 - lse2)
template <typename Tin>
__device__ __forceinline__ void grad_vec(const uint4& xv, float2 cc2, float2 nl, float2 ng, float* o) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(&xv);
  if (sizeof(Tin) == 2) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 z = make_float2(bf16lo(w[j]), bf16hi(w[j]));
      const float2 d = __ffma2_rn(z, cc2, nl);
      const float2 pr = make_float2(ex2(d.x), ex2(d.y));
      const float2 dz = __fmul2_rn(pr, ng);
      o[2 * j] = dz.x;
      o[2 * j + 1] = dz.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float2 z = make_float2(__uint_as_float(w[2 * j]), __uint_as_float(w[2 * j + 1]));
      const float2 d = __ffma2_rn(z, cc2, nl);
      const float2 pr = make_float2(ex2(d.x), ex2(d.y));
      const float2 dz = __fmul2_rn(pr, ng);
      o[2 * j] = dz.x;
      o[2 * j + 1] = dz.y;
    }
  }
}

// store EPV outputs of one full vector (compile-time widths, streaming stores)
template <typename Tout, int EPV>
__device__ __forceinline__ void store_full(uint8_t* dst, const float* o) {
  if (sizeof(Tout) == 2) {
    if (EPV == 8) {
      stg128_cs(dst, make_uint4(pack_bf16x2(o[0], o[1]), pack_bf16x2(o[2], o[3]), pack_bf16x2(o[4], o[5]),
                                pack_bf16x2(o[6], o[7])));
    } else {
      *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16x2(o[0], o[1]), pack_bf16x2(o[2], o[3]));
    }
  } else {
#pragma unroll
    for (int e = 0; e < EPV; e += 4)
      stg128_cs(dst + 4 * e, make_uint4(__float_as_uint(o[e]), __float_as_uint(o[e + 1]), __float_as_uint(o[e + 2]),
                                        __float_as_uint(o[e + 3])));
  }
}

template <typename Tin, int WARPS, int STAGES>
__device__ __forceinline__ void bwd_issue(OCur& pc, const BwdParams& p, uint64_t* bars, uint8_t* ring, int slot,
                                          int lane, uint64_t pol) {
  const int64_t v0 = (int64_t)pc.c * BCH_VEC;
  const int64_t nv = min((int64_t)BCH_VEC, p.nvec - v0);
  if (lane == 0) {
    mbar_arrive_expect_tx(&bars[slot], (uint32_t)nv * 16u);
    bulk_g2s_hint(ring + (size_t)slot * BCH_BYTES, p.logits + pc.t * p.ld_bytes + v0 * 16, (uint32_t)nv * 16u,
                  &bars[slot], pol);
  }
  ocur_advance(pc, p, WARPS);
  ocur_to_kept(pc, p, WARPS);
}

#ifndef DART_BWD_MINB
#define DART_BWD_MINB 1
#endif
// DART_BWD_FULL=1 takes an unpredicated path for full chunks: fewer
// instructions, but measured 14% SLOWER on B200 (6.17 vs 5.41 ms, store
// drain stalls: long_scoreboard on STG source registers + lg_throttle), so
// the per-vector guarded path is the default.
#ifndef DART_BWD_FULL
#define DART_BWD_FULL 0
#endif
// DART_BWD_TMAST=1: bf16 -> bf16 full chunks are written by one bulk
// shared->global copy per 4 KB chunk (TMA store, SASS UBLKCP) from a per-warp
// double-buffered staging area instead of 8 STG.128 per lane; masked chunks
// are bulk-stored from a zero page.  Correct (parity + racecheck/memcheck
// clean) but measured SLOWER on B200: bwd sweep 6.16 vs 5.48 ms (84.6% vs
// 95.1% of the copy peak) -- the staging STS + proxy fence + bulk-group waits
// cost more than the streaming STG.128 they replace.  Off by default.
#ifndef DART_BWD_TMAST
#define DART_BWD_TMAST 0
#endif
// DART_BWD_V8=1: bf16 -> bf16 full chunks (all 256 vectors inside the row, no
// tail) run without per-vector guards and each lane owns PAIRS of adjacent
// 16-byte input vectors, so its 16 gradients leave in one 32-byte store
// (st.global.v8.b32, SASS STG.E.256): 31% fewer instructions than the guarded
// STG.128 path (1.68e9 vs 2.43e9 per launch, ncu) -- and SLOWER on B200:
// 6.07 vs 5.35 ms isolated.  ncu: 26% of warp stalls become long_scoreboard
// on the STG.256 source registers (ptxas reuses them for the next pair's
// unpack right after the store, so each warp waits for the LSU to drain its
// 1 KB store).  =2 spreads the stores (one opaque uniform branch per pair):
// 6.07 ms, same.  DART_BWD_FULL=2 (STG.128, no per-lane guards, spread the
// same way): 6.2 ms.  The guarded path stays the default.  Needs 32-byte
// aligned gradient rows (checked per launch).
#ifndef DART_BWD_V8
#define DART_BWD_V8 0
#endif
__device__ __forceinline__ void stg256_cs(void* p, uint4 a, uint4 b) {
  asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z),
               "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void sts128(void* p, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(p)), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
template <typename Tin, typename Tout, int WARPS, int STAGES>
__global__ void __launch_bounds__(WARPS * 32, DART_BWD_MINB)
bwd_sweep_kernel(const BwdParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int EPV = 16 / sizeof(Tin);       // logits per 16-byte input vector
  constexpr bool OUT_BF16 = sizeof(Tout) == 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + (size_t)warp * STAGES * BCH_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)WARPS * STAGES * BCH_BYTES) + warp * STAGES;
  constexpr bool TMAST = DART_BWD_TMAST && sizeof(Tin) == 2 && sizeof(Tout) == 2;
  constexpr bool V8T = DART_BWD_V8 && !DART_BWD_TMAST && sizeof(Tin) == 2 && sizeof(Tout) == 2;
  const bool v8_ok = V8T && ((p.ldg_bytes & 31) == 0) && ((reinterpret_cast<uintptr_t>(p.dlogits) & 31) == 0);
  // TMA-store staging: [WARPS][2][BCH_BYTES] then one zero page (after the barriers, 1 KB aligned)
  uint8_t* stage_base = smem + (((size_t)WARPS * STAGES * BCH_BYTES + (size_t)WARPS * STAGES * 8 + 1023) & ~(size_t)1023);
  uint8_t* stg_buf = stage_base + (size_t)warp * 2 * BCH_BYTES;
  uint8_t* zero_page = stage_base + (size_t)WARPS * 2 * BCH_BYTES;
  int sbuf = 0;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  if (TMAST) {
    for (int i = threadIdx.x; i < BCH_BYTES / 16; i += blockDim.x) sts128(zero_page + i * 16, make_uint4(0u, 0u, 0u, 0u));
    fence_proxy_async_smem();
    __syncthreads();
  }
  __syncwarp();

  // this CTA's contiguous, cost-balanced chunk range [J0, J1)
  const int64_t total = p.step_cost[p.S_loc];
  const int64_t nb = gridDim.x;
  const int64_t J0 = ordinal_at_cost(p, (total * (int64_t)blockIdx.x) / nb);
  const int64_t J1 = ordinal_at_cost(p, (total * ((int64_t)blockIdx.x + 1)) / nb);
  const int tail_elems = (int)(p.V % EPV);
  const float c2 = p.c2;
  const uint64_t pol = policy_evict_first();
  const int4* rec = reinterpret_cast<const int4*>(p.rec);

  OCur cc;
  cc.jend = J1;
  ocur_seek(cc, p, J0 + warp);
  OCur pc = cc;
  ocur_to_kept(pc, p, WARPS);
#pragma unroll 1
  for (int s = 0; s < STAGES; ++s) {
    if (!pc.valid) break;
    bwd_issue<Tin, WARPS, STAGES>(pc, p, bars, ring, s, lane, pol);
  }

  int slot = 0;
  uint32_t phase = 0;
  int64_t cur_t = -1, pre_t = -1;
  const int64_t nvec = p.nvec, T_loc = p.T_loc, ldg_bytes = p.ldg_bytes;
  uint8_t* const dlog = p.dlogits;
  constexpr int64_t OUTV = EPV * (int64_t)sizeof(Tout);   // output bytes per input vector
  int4 cur = make_int4(0, 0, -1, 0), pre = make_int4(0, 0, -1, 0);

#pragma unroll 1
  while (cc.valid) {
    const int64_t t = cc.t;
    const int64_t v0 = (int64_t)cc.c * BCH_VEC;
    const int nv = (int)min((int64_t)BCH_VEC, nvec - v0);
    // full chunk: all lanes hold BVPL complete vectors (no tail, no predicates)
    const bool full8 = v8_ok && (nv == BCH_VEC) && !(tail_elems && v0 + nv == nvec);
    const bool full = !full8 && DART_BWD_FULL && (nv == BCH_VEC) && !(tail_elems && v0 + nv == nvec);
    uint8_t* orow = dlog + t * ldg_bytes;
    uint8_t* olane = orow + (v0 + lane) * OUTV;    // this lane's first output vector
    if (cc.kept) {
      if (t != cur_t) {
        cur = (t == pre_t) ? pre : rec[t];
        cur_t = t;
        if (t + 1 < T_loc) {       // prefetch the next row's record (hidden behind this row)
          pre = rec[t + 1];
          pre_t = t + 1;
        }
      }
      const float g = __int_as_float(cur.x), nl2 = __int_as_float(cur.y), zy = __int_as_float(cur.w);
      const int32_t y = cur.z;
      mbar_wait(&bars[slot], phase);
      const uint8_t* sp = ring + (size_t)slot * BCH_BYTES;
      const float2 cc2 = make_float2(c2, c2), nl = make_float2(nl2, nl2), ng = make_float2(-g, -g);
      uint4 x[BVPL];
      if (V8T && full8) {       // lane owns vector pairs (lane + 32 k): 32 contiguous bytes each
#pragma unroll
        for (int k = 0; k < BVPL / 2; ++k) {
          x[2 * k] = lds128(sp + (lane + 32 * k) * 32);
          x[2 * k + 1] = lds128(sp + (lane + 32 * k) * 32 + 16);
        }
      } else if (full) {
#pragma unroll
        for (int k = 0; k < BVPL; ++k) x[k] = lds128(sp + (lane + 32 * k) * 16);
      } else {
#pragma unroll
        for (int k = 0; k < BVPL; ++k) {
          const int vi = lane + 32 * k;
          x[k] = (vi < nv) ? lds128(sp + vi * 16) : make_uint4(0u, 0u, 0u, 0u);
        }
      }
      // consume every loaded word before the slot is handed back to the copy
      // engine (read-then-async-write: the reads have completed)
      uint32_t dep = 0;
#pragma unroll
      for (int k = 0; k < BVPL; ++k) dep |= x[k].x | x[k].y | x[k].z | x[k].w;
      asm volatile("" ::"r"(dep));
      __syncwarp();
      if (pc.valid) bwd_issue<Tin, WARPS, STAGES>(pc, p, bars, ring, slot, lane, pol);
      if (++slot == STAGES) { slot = 0; phase ^= 1u; }
      if (V8T && full8) {
#pragma unroll
        for (int k = 0; k < BVPL / 2; ++k) {
          float o[16];
#if DART_BWD_V8 == 2
          // always true on a full chunk, but opaque to the compiler: one branch
          // region per pair keeps each pair's stores next to its math
          if ((nv >> 6) <= k) break;
#endif
          grad_vec<Tin>(x[2 * k], cc2, nl, ng, o);
          grad_vec<Tin>(x[2 * k + 1], cc2, nl, ng, o + 8);
          stg256_cs(orow + (v0 + 2 * (lane + 32 * k)) * 16,
                    make_uint4(pack_bf16x2(o[0], o[1]), pack_bf16x2(o[2], o[3]), pack_bf16x2(o[4], o[5]),
                               pack_bf16x2(o[6], o[7])),
                    make_uint4(pack_bf16x2(o[8], o[9]), pack_bf16x2(o[10], o[11]), pack_bf16x2(o[12], o[13]),
                               pack_bf16x2(o[14], o[15])));
        }
        if (y >= 0) {           // target element g (1 - p_y), after its pair's store (same thread)
          const int64_t yv = y / EPV;
          if (yv >= v0 && yv < v0 + BCH_VEC && lane == (int)(((yv - v0) >> 1) & 31)) {
            const float py = ex2(fmaf(zy, c2, nl2));
            reinterpret_cast<__nv_bfloat16*>(orow)[y] = __float2bfloat16_rn(fmaf(-g, py, g));
          }
        }
        ocur_advance(cc, p, WARPS);
        continue;
      }
      if (TMAST && nv == BCH_VEC && !(tail_elems && v0 + nv == nvec)) {
        // gradient of the chunk into this warp's staging buffer, then one bulk store
        if (lane == 0) bulk_wait_read<1>();         // the buffer's previous bulk store has read it
        __syncwarp();
        uint8_t* sb = stg_buf + (size_t)sbuf * BCH_BYTES;
#pragma unroll
        for (int k = 0; k < BVPL; ++k) {
          float o[EPV];
          grad_vec<Tin>(x[k], cc2, nl, ng, o);
          sts128(sb + (lane + 32 * k) * 16, make_uint4(pack_bf16x2(o[0], o[1]), pack_bf16x2(o[2], o[3]),
                                                       pack_bf16x2(o[4], o[5]), pack_bf16x2(o[6], o[7])));
        }
        if (y >= 0) {                               // target element: g (1 - p_y)
          const int64_t yv = y / EPV;
          if (yv >= v0 && yv < v0 + nv && lane == (int)((yv - v0) & 31)) {
            const float py = ex2(fmaf(zy, c2, nl2));
            reinterpret_cast<__nv_bfloat16*>(sb)[y - v0 * EPV] = __float2bfloat16_rn(fmaf(-g, py, g));
          }
        }
        fence_proxy_async_smem();                   // generic-proxy smem writes -> visible to the bulk copy
        __syncwarp();
        if (lane == 0) {
          bulk_s2g(orow + v0 * OUTV, sb, (uint32_t)BCH_BYTES);
          bulk_commit();
        }
        sbuf ^= 1;
        ocur_advance(cc, p, WARPS);
        continue;
      }
      if (full) {
#pragma unroll
        for (int k = 0; k < BVPL; ++k) {
#if DART_BWD_FULL == 2
          if ((nv >> 5) <= k) break;   // always true here; one branch region per vector (spreads the stores)
#endif
#if DART_BWD_STYLE == 1
          if (lane + 32 * k < nv) {   // always true here: keeps compute/store of each vector together
#endif
          float o[EPV];
#if DART_BWD_STYLE == 2
          if (k > 0) {  // order: store(k-1) before the math of vector k (spreads the stores)
            asm volatile("" : "+r"(x[k].x), "+r"(x[k].y), "+r"(x[k].z), "+r"(x[k].w));
          }
#endif
          grad_vec<Tin>(x[k], cc2, nl, ng, o);
          store_full<Tout, EPV>(olane + k * 32 * OUTV, o);
#if DART_BWD_STYLE == 1
          }
#endif
        }
      } else {
#pragma unroll
        for (int k = 0; k < BVPL; ++k) {
          const int vi = lane + 32 * k;
          if (vi < nv) {
            const int64_t gv = v0 + vi;
            float o[EPV];
            grad_vec<Tin>(x[k], cc2, nl, ng, o);
            const int nvalid = (tail_elems && gv == nvec - 1) ? tail_elems : EPV;
            uint8_t* dst = orow + gv * OUTV;
            if (OUT_BF16) store_vals_bf16(dst, o, nvalid, EPV);
            else store_vals_f32(dst, o, nvalid, EPV);
          }
        }
      }
      // target element: dz_y = g (1 - p_y), written after the vector store (same thread)
      if (y >= 0) {
        const int64_t yv = y / EPV;
        if (yv >= v0 && yv < v0 + nv && lane == (int)((yv - v0) & 31)) {
          const float py = ex2(fmaf(zy, c2, nl2));
          const float dzy = fmaf(-g, py, g);
          if (OUT_BF16) reinterpret_cast<__nv_bfloat16*>(orow)[y] = __float2bfloat16_rn(dzy);
          else reinterpret_cast<float*>(orow)[y] = dzy;
        }
      }
    } else {
      // masked step: zeros, no read
      if (V8T && full8) {
        const uint4 zz = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int k = 0; k < BVPL / 2; ++k) stg256_cs(orow + (v0 + 2 * (lane + 32 * k)) * 16, zz, zz);
        ocur_advance(cc, p, WARPS);
        continue;
      }
      if (TMAST && nv == BCH_VEC && !(tail_elems && v0 + nv == nvec)) {
        if (lane == 0) {
          bulk_s2g(orow + v0 * OUTV, zero_page, (uint32_t)BCH_BYTES);
          bulk_commit();
        }
        ocur_advance(cc, p, WARPS);
        continue;
      }
      float o[EPV];
#pragma unroll
      for (int e = 0; e < EPV; ++e) o[e] = 0.f;
      if (full) {
#pragma unroll
        for (int k = 0; k < BVPL; ++k) store_full<Tout, EPV>(olane + k * 32 * OUTV, o);
      } else {
#pragma unroll
        for (int k = 0; k < BVPL; ++k) {
          const int vi = lane + 32 * k;
          if (vi < nv) {
            const int64_t gv = v0 + vi;
            const int nvalid = (tail_elems && gv == nvec - 1) ? tail_elems : EPV;
            uint8_t* dst = orow + gv * OUTV;
            if (OUT_BF16) store_vals_bf16(dst, o, nvalid, EPV);
            else store_vals_f32(dst, o, nvalid, EPV);
          }
        }
      }
    }
    ocur_advance(cc, p, WARPS);
  }
  if (TMAST && lane == 0) bulk_wait_read<0>();     // smem must outlive the last bulk stores' reads
  if (TMAST) __syncthreads();
}

// ============================================================== launchers
cudaError_t launch_bwd_prep(const BwdPrepParams& p, cudaStream_t st) {
  bwd_prep_kernel<<<1, 1024, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_rowrec(const RowRecParams& p, cudaStream_t st) {
  if (p.T_loc <= 0) return cudaSuccess;
  int64_t blocks = (p.T_loc + 255) / 256;
  if (blocks > 8192) blocks = 8192;
  rowrec_kernel<<<(unsigned)blocks, 256, 0, st>>>(p);
  return cudaGetLastError();
}

template <typename Tin, typename Tout, int WARPS, int STAGES>
static cudaError_t launch_bwd_t(const BwdParams& p, int num_sms, cudaStream_t st) {
  constexpr bool TMAST = DART_BWD_TMAST && sizeof(Tin) == 2 && sizeof(Tout) == 2;
  size_t smem = (size_t)WARPS * STAGES * BCH_BYTES + (size_t)WARPS * STAGES * 8;
  if (TMAST) smem = ((smem + 1023) & ~(size_t)1023) + (size_t)WARPS * 2 * BCH_BYTES + BCH_BYTES + 1024;
  auto kern = bwd_sweep_kernel<Tin, Tout, WARPS, STAGES>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WARPS * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)num_sms * per_sm;
  kern<<<(unsigned)grid, WARPS * 32, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_bwd_sweep(const BwdParams& p, bool in_bf16, bool out_bf16, int num_sms, cudaStream_t st) {
  if (in_bf16 && out_bf16) return launch_bwd_t<__nv_bfloat16, __nv_bfloat16, BWD_WARPS, BWD_STAGES>(p, num_sms, st);
  if (in_bf16) return launch_bwd_t<__nv_bfloat16, float, BWD_WARPS, BWD_STAGES>(p, num_sms, st);
  if (out_bf16) return launch_bwd_t<float, __nv_bfloat16, BWD_WARPS, BWD_STAGES>(p, num_sms, st);
  return launch_bwd_t<float, float, BWD_WARPS, BWD_STAGES>(p, num_sms, st);
}

}  // namespace dart
