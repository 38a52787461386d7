// dart_lmhead.cu -- SURVEY §8(f) NEXT #3: the LM head fused into the loss
// pass, forward and backward.
//
// z_{t,v} = sum_k h_{t,k} W_{v,k} (the logits whose softmax / T is
// pi_theta(a|h,s), Eq. 1) is computed on the 5th-generation
// tensor cores: tcgen05.mma (bf16 x bf16 -> fp32) with both operands staged
// into shared memory by TMA (128-byte swizzle) and the accumulator in TMEM.
// The [T, V] logits never touch memory; the epilogue reads each 128 x 256
// accumulator tile back with tcgen05.ld and
//   forward  (DZ = false): folds it into the per-row online softmax statistics
//            (m, s, u) of the log2 domain (the logits sweep's algebra,
//            PAPER.md:238 entropy) plus the target's logit;
//   backward (DZ = true):  turns it into the loss gradient of the row,
//            dz_v = g_t (delta_{v,y} - 2^(z_v c2 - lse2_t)) (PAPER.md:256-259,
//            g_t = c_s dell_t invT), rounded to bf16 and stored -- the rows are
//            the KEPT rows only (masked steps have no gradient),
//            gathered into a compact block first (lmhead_gather_kernel).
//
// Work item = (128-row block mb, vocabulary chunk nc of LM_NT_PER_CHUNK
// 256-column tiles); in the forward each item leaves one (m, s, u) partial per
// row, folded in chunk order by lmhead_combine_kernel (dart_fwd.cu).
// Persistent CTAs (one per SM) walk the items in a super-column raster:
// LM_GROUP_NC chunks x all row blocks, chunks innermost, so the ~148
// concurrently active items touch ~37 hidden blocks and ~4 weight chunks at a
// time (L2 resident).
//
// Warp roles (192 threads): warp 0 = TMA producer (one lane), warp 1 = TMEM
// allocator + MMA issuer (one lane), warps 2..5 = epilogue (warp w reads TMEM
// lanes 32*(w%4) .. +31, i.e. accumulator rows).  Pipelines: LM_STAGES smem
// stages (full/empty mbarriers), two TMEM accumulators of 256 fp32 columns
// (tfull/tempty), so the epilogue of tile i overlaps the MMAs of tile i+1.
// (A CTA-pair cta_group::2 form was measured slower under the 1 kW power cap,
// DESIGN.md §9, and is not shipped.)
#include <cstdio>
#include <cstdlib>

#include "dart_common.cuh"
#include "dart_internal.h"
#include "dart_tc.cuh"

namespace dart {
namespace {

// 32-byte streaming store (st.global.v8.b32, SASS STG.E.256): dst 32-byte aligned
__device__ __forceinline__ void stg256_cs(void* p, uint4 a, uint4 b) {
  asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z),
               "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}
constexpr int LM_BM = 128, LM_BN = 256, LM_BK = 64, LM_STAGES = 4, LM_ACC = 2;
constexpr int LM_THREADS = 192;
constexpr uint32_t LM_A_BYTES = LM_BM * LM_BK * 2;   // 16 KB
constexpr uint32_t LM_B_BYTES = LM_BN * LM_BK * 2;   // 32 KB
constexpr uint32_t LM_STAGE_BYTES = LM_A_BYTES + LM_B_BYTES;
constexpr size_t LM_SMEM = 1024 + (size_t)LM_STAGES * LM_STAGE_BYTES + 256;
constexpr uint32_t LM_TMEM_COLS = LM_ACC * LM_BN;     // 512: the whole TMEM of the SM
constexpr float LM_MASKED = -1.0e30f;                 // raw logit for columns >= V

using tc::fence_after;
using tc::fence_before;
using tc::tma_load_2d;
using tc::tma_prefetch_desc;
using tc::tmem_ld32;
using tc::umma_commit;

constexpr uint32_t LM_IDESC = tc::idesc_bf16_f32(LM_BM, LM_BN, false, false);

__device__ __forceinline__ uint64_t sw128_kmajor_desc(uint32_t saddr) { return tc::smem_desc_sw128(saddr, 16, 1024); }
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  tc::umma_bf16(tmem_d, da, db, LM_IDESC, accumulate);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) { tc::mbar_arrive1(bar); }
__device__ __forceinline__ void tc_fence_after() { fence_after(); }
__device__ __forceinline__ void tc_fence_before() { fence_before(); }

// work item -> (row block, vocabulary chunk): super-columns of group_nc chunks,
// row blocks outer, chunks inner
__device__ __forceinline__ void lm_item(const LmParams& p, int64_t it, int& mb, int& nc) {
  const int64_t per_sc = (int64_t)p.n_mb * p.group_nc;
  const int sc = (int)(it / per_sc);
  const int rem = (int)(it - (int64_t)sc * per_sc);
  const int gn = min(p.group_nc, p.n_nc - sc * p.group_nc);
  mb = rem / gn;
  nc = sc * p.group_nc + rem % gn;
}

// Rows of the A operand: the forward runs over the shard's T_loc rows; the
// backward over the n_kept gathered rows (a device count: items past it are
// skipped by every role, so the launch needs no host sync).
__device__ __forceinline__ int64_t lm_rows(const LmParams& p) { return p.DZ_n_kept ? *p.DZ_n_kept : p.T_loc; }

template <bool DZ>
__global__ void __launch_bounds__(LM_THREADS, 1)
    lmhead_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const LmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + LM_STAGES * LM_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + LM_STAGES * LM_STAGE_BYTES);
  uint64_t* empty = full + LM_STAGES;
  uint64_t* tfull = empty + LM_STAGES;
  uint64_t* tempty = tfull + LM_ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + LM_ACC);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t unit0 = blockIdx.x, nunits = gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < LM_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < LM_ACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);   // the four epilogue warps
    }
    fence_mbar_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, LM_TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int KB = (p.K + LM_BK - 1) / LM_BK;
  const int64_t M = lm_rows(p);

  if (warp == 0) {
    // ---------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0;
      for (int64_t it = unit0; it < p.n_items; it += nunits) {
        int mb, nc;
        lm_item(p, it, mb, nc);
        if ((int64_t)mb * LM_BM >= M) continue;
        const int nt0 = nc * p.nt_per_chunk, nt1 = min(nt0 + p.nt_per_chunk, p.n_nt);
        for (int nt = nt0; nt < nt1; ++nt) {
          for (int kb = 0; kb < KB; ++kb) {
            mbar_wait(&empty[stage], ph ^ 1u);
            mbar_arrive_expect_tx(&full[stage], LM_STAGE_BYTES);
            tma_load_2d(sA + stage * LM_A_BYTES, &tmA, &full[stage], kb * LM_BK, mb * LM_BM);
            tma_load_2d(sB + stage * LM_B_BYTES, &tmB, &full[stage], kb * LM_BK, nt * LM_BN);
            if (++stage == LM_STAGES) {
              stage = 0;
              ph ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      int stage = 0, acc = 0;
      uint32_t ph = 0, aph = 0;
      for (int64_t it = unit0; it < p.n_items; it += nunits) {
        int mb, nc;
        lm_item(p, it, mb, nc);
        if ((int64_t)mb * LM_BM >= M) continue;
        const int nt0 = nc * p.nt_per_chunk, nt1 = min(nt0 + p.nt_per_chunk, p.n_nt);
        for (int nt = nt0; nt < nt1; ++nt) {
          mbar_wait(&tempty[acc], aph ^ 1u);
          tc_fence_after();
          const uint32_t d_tmem = tmem + (uint32_t)(acc * LM_BN);
          for (int kb = 0; kb < KB; ++kb) {
            mbar_wait(&full[stage], ph);
            tc_fence_after();
            const uint64_t da = sw128_kmajor_desc(smem_u32(sA + stage * LM_A_BYTES));
            const uint64_t db = sw128_kmajor_desc(smem_u32(sB + stage * LM_B_BYTES));
#pragma unroll
            for (int k = 0; k < LM_BK / 16; ++k)   // UMMA_K = 16 bf16 = 32 B along the swizzled row
              umma_bf16(d_tmem, da + (uint64_t)(2 * k), db + (uint64_t)(2 * k), (kb | k) != 0 ? 1u : 0u);
            umma_commit(&empty[stage]);            // frees the smem stage when these MMAs retire
            if (++stage == LM_STAGES) {
              stage = 0;
              ph ^= 1u;
            }
          }
          umma_commit(&tfull[acc]);                // accumulator tile complete
          if (++acc == LM_ACC) {
            acc = 0;
            aph ^= 1u;
          }
        }
      }
    }
  } else {
    // ---------------------------------------------------------- epilogue
    const int q = warp & 3;            // TMEM lane quarter this warp may access
    const int r = q * 32 + lane;       // accumulator row of this thread
    const float c2 = p.c2;
    int acc = 0;
    uint32_t aph = 0;
    for (int64_t it = unit0; it < p.n_items; it += nunits) {
      int mb, nc;
      lm_item(p, it, mb, nc);
      if ((int64_t)mb * LM_BM >= M) continue;
      const int nt0 = nc * p.nt_per_chunk, nt1 = min(nt0 + p.nt_per_chunk, p.n_nt);
      const int64_t row = (int64_t)mb * LM_BM + r;
      const bool valid = row < M;
      // forward state
      float m_run = LM_MASKED;         // running max of z*c2 (log2 units); any real logit exceeds it
      double S = 0.0, U = 0.0;         // sum 2^(x-m), sum 2^(x-m)(x-m)
      float zy = 0.0f;
      // backward row record {g, -lse2, y, local row}
      int4 rr = make_int4(0, 0, -1, 0);
      if (DZ && valid) rr = reinterpret_cast<const int4*>(p.DZ_rec)[row];
      const int64_t y = DZ ? (int64_t)rr.z : (valid ? (int64_t)p.target[row] : -1);
      uint8_t* const orow = DZ ? p.DZ_out + row * p.DZ_ldg_bytes : nullptr;
      for (int nt = nt0; nt < nt1; ++nt) {
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * LM_BN);
#pragma unroll 1
        for (int j = 0; j < LM_BN / 32; ++j) {
          float x[32];
          tmem_ld32(tbase + (uint32_t)(j * 32), x);
          const int64_t col0 = (int64_t)nt * LM_BN + j * 32;
          if (DZ) {
            // dz_v = -g 2^(z_v c2 - lse2) for v != y, g (1 - p_y) at the target
            if (!valid || col0 >= p.V) continue;
            const float g = __int_as_float(rr.x), nl2 = __int_as_float(rr.y);
            const int jy = (int)(y - col0);   // in [0, 32) iff the target is in this group
            uint32_t o[16];
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const float p0 = ex2(fmaf(x[i], c2, nl2)), p1 = ex2(fmaf(x[i + 1], c2, nl2));
              const float d0 = (i == jy) ? fmaf(-g, p0, g) : -g * p0;
              const float d1 = (i + 1 == jy) ? fmaf(-g, p1, g) : -g * p1;
              o[i / 2] = pack_bf16x2(d0, d1);
            }
            uint8_t* dst = orow + col0 * 2;
            if (col0 + 32 <= p.V) {
              if (p.DZ_st256) {       // 32-byte aligned rows: two STG.256 (measured 5% faster than four STG.128)
                stg256_cs(dst, make_uint4(o[0], o[1], o[2], o[3]), make_uint4(o[4], o[5], o[6], o[7]));
                stg256_cs(dst + 32, make_uint4(o[8], o[9], o[10], o[11]), make_uint4(o[12], o[13], o[14], o[15]));
              } else {
                stg128_cs(dst, make_uint4(o[0], o[1], o[2], o[3]));
                stg128_cs(dst + 16, make_uint4(o[4], o[5], o[6], o[7]));
                stg128_cs(dst + 32, make_uint4(o[8], o[9], o[10], o[11]));
                stg128_cs(dst + 48, make_uint4(o[12], o[13], o[14], o[15]));
              }
            } else {                        // vocabulary tail
              const int nv = (int)(p.V - col0);
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (i < nv)
                  reinterpret_cast<uint16_t*>(dst)[i] = (uint16_t)((i & 1) ? (o[i / 2] >> 16) : (o[i / 2] & 0xffffu));
            }
            continue;
          }
          if (col0 + 32 > p.V) {       // vocabulary tail (TMA zero-filled columns >= V)
            const int nv = (int)max((int64_t)0, p.V - col0);
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = (i < nv) ? x[i] : LM_MASKED;
          }
          float mx = x[0];
#pragma unroll
          for (int i = 1; i < 32; ++i) mx = fmaxf(mx, x[i]);
          const float gm = mx * c2;
          if (gm > m_run) {              // exact rescale of (S, U) to the new max
            const float dm = m_run - gm;
            const double f = (double)ex2(dm);
            U = f * (U + S * (double)dm);
            S *= f;
            m_run = gm;
          }
          float s0 = 0.f, s1 = 0.f, u0 = 0.f, u1 = 0.f;
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float d0 = fmaf(x[i], c2, -m_run), d1 = fmaf(x[i + 1], c2, -m_run);
            const float e0 = ex2(d0), e1 = ex2(d1);
            s0 += e0;
            s1 += e1;
            u0 = fmaf(e0, d0, u0);
            u1 = fmaf(e1, d1, u1);
          }
          S += (double)(s0 + s1);
          U += (double)(u0 + u1);
          const int64_t jy = y - col0;
          if ((uint64_t)jy < 32u) {
            // binary select tree on the bits of jy (a plain x[jy] would put x in local memory)
            float t[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) t[i] = (jy & 16) ? x[i + 16] : x[i];
#pragma unroll
            for (int i = 0; i < 8; ++i) t[i] = (jy & 8) ? t[i + 8] : t[i];
#pragma unroll
            for (int i = 0; i < 4; ++i) t[i] = (jy & 4) ? t[i + 4] : t[i];
#pragma unroll
            for (int i = 0; i < 2; ++i) t[i] = (jy & 2) ? t[i + 2] : t[i];
            zy = (jy & 1) ? t[1] : t[0];
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (++acc == LM_ACC) {
          acc = 0;
          aph ^= 1u;
        }
      }
      if (!DZ && valid) {
        const int64_t idx = row * p.n_nc + nc;
        p.part_m[idx] = m_run;
        p.part_s[idx] = S;
        p.part_u[idx] = U;
        if (y >= (int64_t)nt0 * LM_BN && y < (int64_t)nt1 * LM_BN) p.zy[row] = zy;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tc::tmem_dealloc(tmem, LM_TMEM_COLS);
  }
}

// Backward gather (K_lm_g): the kept rows of the shard, in row order, into a
// compact block -- row i of the block is local row t with
// i = kept_off[s(t)] + (t - t0(s)) (kept_off = the exclusive prefix of kept
// tokens over the local steps, bwd_prep's step_cost with unit costs) -- with
// its 16-byte record {g = c_s dell_t invT, -lse2_t, y_t, t} and its hidden
// state (one warp per row, 16-byte vectors).
__global__ void lmhead_gather_kernel(const LmGatherParams p) {
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < p.T_loc; t += warps) {
    const int32_t s = p.tok_step[t];
    if (!p.keep[p.step_begin + s]) continue;
    const int64_t t0 = p.step_tok_off[p.step_begin + s] - p.tok_begin;
    const int64_t i = p.kept_off[s] + (t - t0);
    if (lane == 0) {
      int4 r;
      r.x = __float_as_int((float)(p.step_scale[s] * (double)p.dell[t] * p.invT));
      r.y = __float_as_int(-p.lse2[t]);
      const int32_t y = p.target[t];
      r.z = (y >= 0 && y < p.V) ? y : -1;
      r.w = (int32_t)t;
      reinterpret_cast<int4*>(p.rec)[i] = r;
      p.kept_rows[i] = (int32_t)t;
    }
    const uint4* src = reinterpret_cast<const uint4*>(p.hidden + t * p.ld_h * 2);
    uint4* dst = reinterpret_cast<uint4*>(p.hidden_kept + i * p.ld_hk * 2);
    for (int64_t v = lane; v < p.d / 8; v += 32) dst[v] = src[v];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *p.n_kept = p.kept_off[p.S_loc];
}

}  // namespace

cudaError_t launch_lmhead(const void* hidden, int64_t ld_h, const void* weight, int64_t ld_w, const LmParams& p,
                          int num_sms, cudaStream_t st) {
  if (p.T_loc <= 0 || p.n_items <= 0) return cudaSuccess;
  CUtensorMap tmA, tmB;
  if (!tc::make_map_bf16(&tmA, hidden, p.T_loc, p.K, ld_h, LM_BK, LM_BM)) return cudaErrorInvalidValue;
  if (!tc::make_map_bf16(&tmB, weight, p.V, p.K, ld_w, LM_BK, LM_BN)) return cudaErrorInvalidValue;
  const bool dz = p.DZ_n_kept != nullptr;
  auto kern = dz ? lmhead_kernel<true> : lmhead_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LM_SMEM);
  if (e != cudaSuccess) return e;   // (per call: the attribute is per device)
  const int64_t grid = p.n_items < num_sms ? p.n_items : num_sms;
  kern<<<(unsigned)grid, LM_THREADS, LM_SMEM, st>>>(tmA, tmB, p);
  return cudaGetLastError();
}

cudaError_t launch_lmhead_gather(const LmGatherParams& p, cudaStream_t st) {
  int64_t blocks = (p.T_loc + 7) / 8;
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) blocks = 1;
  lmhead_gather_kernel<<<(unsigned)blocks, 256, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace dart
