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
    // dart_stats is NV doubles in field order (loss, n_tok, n_kept_tok, n_kept_step, sum_clip,
    // sum_trunc, sum_w, sum_adv, sum_adv2, sum_H, sum_kl)
    double* o = reinterpret_cast<double*>(p.stats);
#pragma unroll
    for (int i = 0; i < NV; ++i) o[i] = p.accumulate ? o[i] + tot[i] : tot[i];
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
constexpr int BVPL = BCH_VEC / 32;
   // 16-byte vectors per lane per bwd chunk
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

// The sweep's code shape is part of its performance: every
// 16-byte input vector's gradient is computed and stored inside its own
// guarded region, so the eight 128-bit stores of a chunk leave interleaved
// with the math (an unguarded loop bursts them and stalls on the store queue;
// wider 32-byte stores and TMA bulk stores from shared memory were both
// measured slower).  Hoisting the per-vector address / tail arithmetic to a
// per-chunk lane base (fewer instructions) also measured slower on B200:
// 6.05 vs 5.74 ms on one box, A/B in one session (profiles/r02_bwd_ab.md).
template <typename Tin, typename Tout, int WARPS, int STAGES>
__global__ void __launch_bounds__(WARPS * 32, 1)
bwd_sweep_kernel(const BwdParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int EPV = 16 / sizeof(Tin);       // logits per 16-byte input vector
  constexpr bool OUT_BF16 = sizeof(Tout) == 2;
  constexpr int OUTV = EPV * (int)sizeof(Tout);   // output bytes per input vector
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + (size_t)warp * STAGES * BCH_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)WARPS * STAGES * BCH_BYTES) + warp * STAGES;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
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
  int4 cur = make_int4(0, 0, -1, 0), pre = make_int4(0, 0, -1, 0);

#pragma unroll 1
  while (cc.valid) {
    const int64_t t = cc.t;
    const int64_t v0 = (int64_t)cc.c * BCH_VEC;
    const int nv = (int)min((int64_t)BCH_VEC, nvec - v0);
    uint8_t* const orow = dlog + t * ldg_bytes;
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
#pragma unroll
      for (int k = 0; k < BVPL; ++k) {
        const int vi = lane + 32 * k;
        x[k] = (vi < nv) ? lds128(sp + vi * 16) : make_uint4(0u, 0u, 0u, 0u);
      }
      fence_reads_before_refill();
      __syncwarp();
      if (pc.valid) bwd_issue<Tin, WARPS, STAGES>(pc, p, bars, ring, slot, lane, pol);
      if (++slot == STAGES) { slot = 0; phase ^= 1u; }
      {
#pragma unroll
        for (int k = 0; k < BVPL; ++k) {
          const int vi = lane + 32 * k;
          if (vi < nv) {
            const int64_t gv = v0 + vi;
            float o[EPV];
            grad_vec<Tin>(x[k], cc2, nl, ng, o);
            const int nvalid = (tail_elems && gv == nvec - 1) ? tail_elems : EPV;
            uint8_t* dst = orow + gv * (int64_t)OUTV;
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
      float o[EPV];
#pragma unroll
      for (int e = 0; e < EPV; ++e) o[e] = 0.f;
#pragma unroll
      for (int k = 0; k < BVPL; ++k) {
        const int vi = lane + 32 * k;
        if (vi < nv) {
          const int64_t gv = v0 + vi;
          const int nvalid = (tail_elems && gv == nvec - 1) ? tail_elems : EPV;
          uint8_t* dst = orow + gv * (int64_t)OUTV;
          if (OUT_BF16) store_vals_bf16(dst, o, nvalid, EPV);
          else store_vals_f32(dst, o, nvalid, EPV);
        }
      }
    }
    ocur_advance(cc, p, WARPS);
  }
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
  const size_t smem = (size_t)WARPS * STAGES * BCH_BYTES + (size_t)WARPS * STAGES * 8;
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
